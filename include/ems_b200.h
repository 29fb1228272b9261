/*
 * ems_b200.h -- C ABI of the B200-native EMS prefill-compress path.
 *
 * This is the drop-in boundary for the reference's prefill hot path
 * (SURVEY.md section 8b).  The reference binds these operations as C++
 * functions on fp64 per-head matrices; here they are batched, stream-ordered,
 * device-pointer entry points over contiguous [B][H][L][d] tensors, so each
 * (b, h) slice is byte-for-byte a reference `Matrix` (proj/include/ems/types.hpp:13-34)
 * in fp32 or bf16.  include/ems_b200/ems.hpp restores the reference's C++
 * signatures (same names, argument order and exceptions, plus a trailing dtype
 * argument where the device precision is selectable) on top of this ABI;
 * INTEGRATION.md shows the bindings.
 *
 *   reference entry point (file:line)                          replaced by
 *   ---------------------------------------------------------  -------------------------
 *   prefill_attention   proj/include/ems/scoring.hpp:52-54      ems_score (out_o != NULL)
 *   prefill_scores      proj/include/ems/scoring.hpp:48-49      ems_score (out_o == NULL)
 *   global/local_score_prefill  scoring.hpp:40-45               ems_score
 *   combine_glo_loc + effective_score  scoring.hpp:58,66        ems_select (prologue)
 *   init_score_state    scoring.hpp:70                          implicit: loc -> loc_past
 *   effective_score     scoring.hpp:66                          ems_effective_score
 *   partition_tokens    proj/include/ems/compressor.hpp:14-25   ems_select (fused) / ems_partition
 *   redundancy_cross    proj/include/ems/analysis.hpp:19-20     ems_redundancy_cross / ems_merge
 *   assign_merge_destinations  compressor.hpp:29               ems_merge (fused) /
 *                                                              ems_assign_merge_destinations
 *   weighted_merge      compressor.hpp:32-51                    ems_compact (fused) / ems_weighted_merge
 *   compress_prefill    compressor.hpp:58-60                    ems_select+ems_merge+ems_compact
 *   engine prefill (score -> compress)  proj/src/engine.cpp:42-82  ems_prefill_compress
 *   engine prefill incl. RoPE           proj/src/engine.cpp:42-82  ems_prefill (raw Q/K)
 *   engine prefill from host matrices   proj/src/engine.cpp:42-82  ems_prefill_host
 *   apply_rope / detail::rotate         proj/src/rope.cpp:10-37    ems_rope
 *   decode_step + decode_update         engine.cpp:150-210, compressor.cpp:244-398  ems_decode_step
 *
 * Conventions
 *  - A "unit" is one (b, h_kv) with its G = heads_q / heads_kv query heads;
 *    unit u = b * heads_kv + h_kv.  Units are independent (no collective).
 *  - All pointers are caller-owned device memory; nothing is allocated inside
 *    the hot path.  Query ems_workspace_bytes() once and pass a workspace of
 *    at least that size (16-byte aligned).  Calls are asynchronous on `stream`.
 *  - Inputs are pre-rotated Q/K for scoring and raw (pre-RoPE) K plus V for the
 *    merge (contract D3).
 *  - GQA (contract D2): per-unit glo/loc are the MEAN over the unit's G query
 *    heads of each head's column sums.
 *  - Status codes mirror the reference's exceptions (proj/include/ems/errors.hpp):
 *    std::invalid_argument -> EMS_INVALID_ARGUMENT, DegenerateInputError ->
 *    EMS_DEGENERATE_INPUT, CorruptionError -> EMS_CORRUPTION.  Host-detectable
 *    errors return immediately; data-dependent ones (zero global mass, LUT
 *    integrity) are recorded in the workspace and returned by ems_sync_status().
 *  - Reentrant: no global mutable state except the thread-local error string.
 */
#ifndef EMS_B200_H
#define EMS_B200_H

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMS_B200_ABI_VERSION 3

#if defined(__GNUC__)
#define EMS_API __attribute__((visibility("default")))
#else
#define EMS_API
#endif

typedef enum {
    EMS_OK = 0,
    EMS_INVALID_ARGUMENT = 1,
    EMS_DEGENERATE_INPUT = 2,
    EMS_CORRUPTION = 3,
    EMS_CUDA_ERROR = 4,
    EMS_UNSUPPORTED = 5,
} ems_status;

typedef enum { EMS_F32 = 0, EMS_BF16 = 1 } ems_dtype;

/* Score-pass implementation.  AUTO picks the tcgen05 kernels for bf16 with
 * head_dim 128 and the SIMT kernels otherwise (fp32 has no tcgen05 MMA kind
 * that keeps the 1e-4 contract; SURVEY.md section 7 "fp32 config 1"). */
typedef enum { EMS_SCORE_AUTO = 0, EMS_SCORE_SIMT = 1, EMS_SCORE_TCGEN05 = 2 } ems_score_impl;

/* Prefill policy (PolicyHandle, proj/include/ems/policies.hpp:12-20; policy_prefill_compress,
 * proj/src/policies.cpp:131-180).  The baselines reuse the select and compact kernels:
 * FULL keeps every token (locals capacity becomes seq_len), STREAMING keeps sink_count
 * sinks plus the most recent tokens, H2O the top-(n_budget - l_win) candidates by glo,
 * SNAPKV the top ones by mean-pooled loc; none of them merges (no TBM set, LUT = kept
 * centers self-mapped).  Numbered so that a zero-initialised descriptor means EMS. */
typedef enum {
    EMS_POLICY_EMS = 0,
    EMS_POLICY_FULL = 1,
    EMS_POLICY_STREAMING = 2,
    EMS_POLICY_H2O = 3,
    EMS_POLICY_SNAPKV = 4,
} ems_policy;

/* Problem descriptor: shapes + CompressionConfig (proj/include/ems/cache.hpp:20-39) + policy. */
typedef struct {
    int32_t batch;
    int32_t heads_q;
    int32_t heads_kv;        /* heads_q % heads_kv == 0 */
    int32_t seq_len;         /* L: prompt tokens */
    int32_t head_dim;        /* d: even, <= 128 (SIMT) / == 128 (tcgen05) */
    int32_t dtype;           /* ems_dtype of Q/K/V, O and the cache K/V */
    int32_t l_win;           /* CompressionConfig::l_win (scores use min(l_win, L)) */
    int32_t n_budget;        /* CompressionConfig::n_budget */
    double tau;              /* merge threshold in [0, 1] */
    double gamma;            /* merge magnification >= 1 */
    int32_t kernel_size;     /* odd pooling window */
    int32_t zero_class;      /* 1: EvictionRealization::zero_class, 0: explicit_removal */
    int32_t key_only;        /* 0: R = cos_k*cos_v (reference); 1: key cosine only (D1) */
    int32_t score_impl;      /* ems_score_impl */
    int64_t first_position;  /* logical position of token 0 */
    int32_t policy;          /* ems_policy (0 = EMS) */
    int32_t sink_count;      /* PolicyHandle::sink_count (streaming_llm; reference default 4) */
    int32_t position_mode;   /* decode expansion RoPE: 0 with_pos (entry position), 1 without_pos
                                (center position); CompressionConfig::position_mode, cache.hpp:11 */
} ems_desc;

/* Per-unit capacities of the compressed cache (fixed-size SoA). */
typedef struct {
    int32_t units;
    int32_t centers;   /* n_budget - l_win */
    int32_t locals;    /* n_budget (keep-all path stores up to n_budget tokens); seq_len for FULL */
    int32_t lut;       /* centers + tbm */
    int32_t tbm;       /* floor((gamma - 1) * n_budget) for EMS, 0 for the baselines */
} ems_cache_dims;

/* The compressed per-unit cache, device SoA (flattened HeadCacheState,
 * proj/include/ems/cache.hpp:41-111).  [u][...] with the capacities above.
 * Keys/values in the desc dtype; scores fp32 triples (glo, loc_past, loc_cur). */
typedef struct {
    void* center_key;       /* [u][centers][d] unit-norm key (slot order = position order) */
    float* center_norm;     /* [u][centers]    preserved key norm */
    void* center_value;     /* [u][centers][d] */
    int32_t* center_pos;    /* [u][centers] */
    float* center_score;    /* [u][centers][3] */
    void* local_key;        /* [u][locals][d]  raw key */
    void* local_value;      /* [u][locals][d] */
    int32_t* local_pos;     /* [u][locals] */
    float* local_score;     /* [u][locals][3] */
    int32_t* lut_pos;       /* [u][lut] sorted by position */
    int32_t* lut_slot;      /* [u][lut] center slot, -1 = zero class */
    int32_t* counts;        /* [u][4] = n_centers, n_locals, n_lut, compressed */
} ems_cache;

/* Intermediate per-unit buffers shared by the staged entry points. */
typedef struct {
    float* pooled;        /* [u][L]  effective score (combine + mean-pool), fp32 */
    int8_t* cls;          /* [u][L]  0 irrelevant, 1 to-be-merged, 2 important, 3 local */
    int32_t* imp_idx;     /* [u][centers] important token indices, ascending (slot order) */
    int32_t* tbm_idx;     /* [u][tbm]     TBM token indices, ascending */
    int32_t* part_counts; /* [u][4] = n_imp, n_tbm, n_irrelevant, n_local */
    int32_t* dest;        /* [u][tbm]     merge destination slot or -1 (zero class) */
} ems_stage;

EMS_API int ems_abi_version(void);
EMS_API const char* ems_last_error(void);
EMS_API const char* ems_status_string(int status);

EMS_API int ems_validate(const ems_desc* desc);
EMS_API int ems_cache_dims_for(const ems_desc* desc, ems_cache_dims* out);
EMS_API size_t ems_workspace_bytes(const ems_desc* desc);

/* (1) Score pass: causal attention O (optional) plus GQA-mean column sums.
 *   q_rot [B][Hq][L][d], k_rot/v [B][Hkv][L][d]  (dtype)
 *   out_o [B][Hq][L][d] (dtype, may be NULL -> score only; v may then be NULL)
 *   lse   [B][Hq][L] fp32 natural-log row log-sum-exp (may be NULL)
 *   glo, loc [B][Hkv][L] fp32 */
EMS_API int ems_score(const ems_desc* desc, const void* q_rot, const void* k_rot, const void* v,
              void* out_o, float* lse, float* glo, float* loc, void* workspace,
              size_t workspace_bytes, cudaStream_t stream);

/* (2) Select: align + combine + pool + radix top-k + classify + index lists. */
EMS_API int ems_select(const ems_desc* desc, const float* glo, const float* loc, const ems_stage* stage,
               void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* partition_tokens (proj/include/ems/compressor.hpp:25, compressor.cpp:48-74) on CALLER pooled
 * scores: pooled [units][L] fp32 -> the stage's class bytes, ascending important / TBM index
 * lists and counts (stage->pooled receives a copy).  The (score desc, index asc) order of the
 * reference's stable sort is exact; ties are decided on the fp32 values.  Needs L > l_win. */
EMS_API int ems_partition(const ems_desc* desc, const float* pooled, const ems_stage* stage, void* workspace,
                          size_t workspace_bytes, cudaStream_t stream);

/* effective_score (proj/include/ems/scoring.hpp:66, scoring.cpp:146-152): mean_pool_1d(
 * combine_glo_loc(glo, loc_past + loc_cur), kernel) for `units` rows of length L (loc_cur may be
 * NULL = zeros), fp64 arithmetic on fp32 scores.  kernel odd and <= L (numerics.cpp:63-68).
 * Zero global mass -> EMS_DEGENERATE_INPUT via ems_sync_status(NULL, workspace, stream);
 * workspace >= 16 bytes. */
EMS_API int ems_effective_score(int32_t units, int32_t L, int32_t kernel, const float* glo, const float* loc_past,
                                const float* loc_cur, float* pooled, void* workspace, size_t workspace_bytes,
                                cudaStream_t stream);

/* assign_merge_destinations (compressor.hpp:29, compressor.cpp:76-95): per row of r [n_rows][n_cols]
 * (fp32) the argmax column (strictly greater wins, so ties go to the lower column) when it reaches
 * tau, else -1 (kZeroClass) -> dest [n_rows]. */
EMS_API int ems_assign_merge_destinations(int32_t n_rows, int32_t n_cols, const float* r, double tau,
                                          int32_t* dest, cudaStream_t stream);

/* weighted_merge (compressor.hpp:46-51, compressor.cpp:97-161) on fp64 device arrays: center
 * column c (unit key [d], value [d], score triple, weight) absorbs the TBM rows i with dest[i] == c
 * in ascending i: ws = w_c + sum w_i; key <- normalize((w_c/ws) u_c + sum (w_i/ws) k_i/|k_i|)
 * (unchanged when that is zero), value <- (w_c/ws) v_c + sum (w_i/ws) v_i, score += member
 * triples; uniform weights when ws <= 0.  Columns without members are untouched.  The LUT
 * entries are the caller's (include/ems_b200/ems.hpp appends them as the reference does). */
EMS_API int ems_weighted_merge(int32_t d, int32_t n_cols, double* center_unit_key, double* center_value,
                               double* center_score, const double* center_weight, int32_t n_tbm,
                               const double* tbm_key, const double* tbm_value, const double* tbm_weight,
                               const double* tbm_score, const int32_t* dest, cudaStream_t stream);

/* (3) Merge assignment: R = cos_k*cos_v (TBM x centers) on raw K/V, argmax with
 * ties to the lower column, tau threshold -> stage->dest. */
EMS_API int ems_merge(const ems_desc* desc, const void* k_raw, const void* v, const ems_stage* stage,
              void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* (4) Compact: centers (unit key, norm, value, position, scores), weighted merge
 * of TBM members into their centers, locals, position-sorted LUT. */
EMS_API int ems_compact(const ems_desc* desc, const void* k_raw, const void* v, const float* glo,
                const float* loc, const ems_stage* stage, const ems_cache* cache,
                void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Whole path (1)-(4); stage may be NULL (then workspace-backed). */
EMS_API int ems_prefill_compress(const ems_desc* desc, const void* q_rot, const void* k_rot,
                         const void* k_raw, const void* v, void* out_o, float* lse, float* glo,
                         float* loc, const ems_stage* stage, const ems_cache* cache,
                         void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Rotary position embedding, detail::rotate (proj/src/rope.cpp:10-28) applied per token as
 * rotate_block does (proj/src/engine.cpp:14-22): x, y [planes][seq_len][head_dim] (dtype),
 * token l at position first_position + l, pair (2i, 2i+1) rotated by pos * base^(-2i/d) in
 * fp64 and rounded once to dtype.  x == y (in place) is allowed. */
EMS_API int ems_rope(int32_t dtype, int32_t planes, int32_t seq_len, int32_t head_dim, double base,
             int64_t first_position, const void* x, void* y, cudaStream_t stream);

/* engine::prefill (proj/src/engine.cpp:42-82) on RAW inputs: RoPE of q [B][Hq][L][d] and
 * k [B][Hkv][L][d] (base rope_base, positions first_position + i; rope_base == 0 means no
 * RoPE) into the caller's q_rot / k_rot scratch (same shapes, may be NULL when rope_base == 0),
 * then the whole path of ems_prefill_compress with k as the raw (pre-RoPE) keys. */
EMS_API int ems_prefill(const ems_desc* desc, double rope_base, const void* q, const void* k,
                const void* v, void* q_rot, void* k_rot, void* out_o, float* lse, float* glo,
                float* loc, const ems_stage* stage, const ems_cache* cache, void* workspace,
                size_t workspace_bytes, cudaStream_t stream);

/* engine::prefill from HOST memory -- the reference's own calling convention (per-head host
 * matrices in, PrefillResult.per_head outputs and the head caches out; proj/src/engine.cpp:42-82,
 * proj/include/ems/engine.hpp:36-45), batched.  h_* are pinned host [B][H][L][d] tensors; d_* are
 * the caller's device staging buffers of the same shapes.  The units are split into `chunks`
 * contiguous groups of geometrically growing size (U/2^(chunks-1), ..., U/4, U/2 units, so compute
 * starts after a small first copy): the host-to-device copy of group c+1 (on copy_stream, or a
 * library-owned per-thread stream when NULL) overlaps the compute of group c (on stream), and each
 * group's results go back as soon as it is done: its compressed cache to h_cache (pinned host SoA
 * with the device cache's shapes; may be NULL) and its attention output rows to h_out_o (pinned
 * host [B][Hq][L][d]; may be NULL, needs out_o).  rope_base > 0: h_q/h_k are raw and RoPE runs on
 * the device into d_q_rot/d_k_rot (h_k_raw/d_k_raw unused); rope_base == 0: h_q/h_k are
 * pre-rotated and h_k_raw/d_k_raw carry the raw keys.  Asynchronous: on return -- on success and
 * on every error after the first enqueue -- `stream` is ordered after every copy and the second
 * compute stream, so synchronising it completes the call. */
/* Workspace that lets ems_prefill_host keep two unit groups in flight (odd groups on a second,
 * library-owned stream with the second part of the workspace) and compute the RoPE (cos, sin)
 * table once for every group (the last part); with ems_workspace_bytes() the groups run one at a
 * time on `stream` and every RoPE launch evaluates its own sines. */
EMS_API size_t ems_prefill_host_workspace_bytes(const ems_desc* desc);
EMS_API int ems_prefill_host(const ems_desc* desc, double rope_base, const void* h_q, const void* h_k,
                     const void* h_k_raw, const void* h_v, void* d_q, void* d_k, void* d_k_raw,
                     void* d_v, void* d_q_rot, void* d_k_rot, void* out_o, void* h_out_o, float* lse,
                     float* glo, float* loc, const ems_cache* d_cache, const ems_cache* h_cache,
                     int32_t chunks, void* workspace, size_t workspace_bytes, cudaStream_t stream,
                     cudaStream_t copy_stream);

/* ---------------------------------------------------------------- decode
 * The EMS decode loop, decode_step (proj/src/engine.cpp:150-210) with decode_update
 * (proj/src/compressor.cpp:376-398), one CTA per unit per step.  The per-unit state is a
 * fixed-capacity device SoA (HeadCacheState, proj/include/ems/cache.hpp:81-111): center
 * slots (slot_alive marks live std::optional slots; a freed slot is reused lowest-first), a
 * ring buffer of exact locals, the position-sorted LUT, and meta[8] = {ring head, locals,
 * LUT entries, window_fill, compressed, live centers, error code, 0}.  Keys/values fp32, scores fp64.
 * Every policy's decode rule (policy_decode_compress, proj/src/policies.cpp:182-242): EMS
 * decode_update; SnapKV graduates locals (decode tokens accumulate); H2O graduates and drops
 * the lowest-glo center; StreamingLLM graduates and drops the oldest non-sink center; full
 * keeps every token. */
typedef struct {
    float* slot_key;      /* [u][slots][d] unit-norm raw key */
    float* slot_norm;     /* [u][slots] */
    float* slot_value;    /* [u][slots][d] */
    int32_t* slot_pos;    /* [u][slots] */
    double* slot_score;   /* [u][slots][3] glo, loc_past, loc_cur */
    int32_t* slot_alive;  /* [u][slots] */
    float* local_key;     /* [u][locals][d] raw key (ring) */
    float* local_value;   /* [u][locals][d] */
    int32_t* local_pos;   /* [u][locals] */
    double* local_score;  /* [u][locals][3] */
    int32_t* lut_pos;     /* [u][lut] */
    int32_t* lut_slot;    /* [u][lut], -1 = zero class */
    int32_t* meta;        /* [u][8] */
} ems_decode_state;

typedef struct {
    int32_t units;
    int32_t slots;   /* center_capacity + 1 (SnapKV: + decode horizon; full: 1) */
    int32_t locals;  /* max(l_win, n_budget) + 1 (full: the whole prompt + decode horizon + 1) */
    int32_t lut;     /* EMS: lut_capacity = floor(gamma * n_budget) (cache.hpp:36-38); else slots */
    int32_t rows;    /* lut + locals: the most expanded rows one step can attend */
} ems_decode_dims;

/* max_positions = the RoPE table size = seq_len + the decode horizon (SnapKV and full grow). */
EMS_API int ems_decode_dims_for(const ems_desc* desc, int32_t max_positions, ems_decode_dims* out);
EMS_API size_t ems_decode_workspace_bytes(const ems_desc* desc, int32_t max_positions);

/* (cos, sin) of position * base^(-2i/d) for positions [0, max_positions), fp64 rounded to
 * fp32: table = float2 [max_positions][head_dim / 2] (device).  Shared by all decode steps. */
EMS_API int ems_rope_table(int32_t head_dim, double base, int32_t max_positions, void* table,
                   cudaStream_t stream);

/* Decode state from a prefill cache (ems_prefill / ems_prefill_compress output); window_fill
 * starts at 0 as engine::prefill leaves it (engine.cpp:74). */
EMS_API int ems_decode_init(const ems_desc* desc, int32_t max_positions, const ems_cache* cache,
                    const ems_decode_state* state, cudaStream_t stream);

/* One decode step for every unit at logical `position` (engine::next_position):
 *   q [B][Hq][d], k / v [B][Hkv][d] raw (pre-RoPE), dtype -> out [B][Hq][d] (dtype),
 *   argmax_position [B][Hq] int32 (logical position of each query head's largest weight).
 * position < max_positions of the RoPE table. */
EMS_API int ems_decode_step(const ems_desc* desc, int64_t position, const void* rope_table,
                    int32_t max_positions, const void* q, const void* k, const void* v, void* out,
                    int32_t* argmax_position, const ems_decode_state* state, void* workspace,
                    size_t workspace_bytes, cudaStream_t stream);

/* Synchronises `stream` and returns the first unit's decode error (EMS_CORRUPTION: stepped past the
 * capacity the state was sized for -- more steps than max_positions - seq_len -- or no free center
 * slot), recorded in meta[6] by the step kernel; a failed unit stops updating. */
EMS_API int ems_decode_sync_status(const ems_desc* desc, const ems_decode_state* state, cudaStream_t stream);

/* Standalone redundancy_cross (analysis.hpp:19-20) for one pair of token groups:
 * k_rows/v_rows [n_rows][d], k_cols/v_cols [n_cols][d] (dtype) -> r [n_rows][n_cols] fp32. */
EMS_API int ems_redundancy_cross(int32_t dtype, int32_t d, const void* k_rows, const void* v_rows,
                         int32_t n_rows, const void* k_cols, const void* v_cols, int32_t n_cols,
                         int32_t key_only, float* r, cudaStream_t stream);

/* analyze_trace's per-head diagnostics (proj/src/experiment.cpp:133-150) for `units`
 * independent token sequences of length L; workspace >= ems_diagnostics_workspace_bytes(units,
 * L); data-dependent errors are read back with ems_sync_status(NULL, workspace, stream).
 *   ems_sparsity_rate:   sparsity_rate(combine_glo_loc(glo, loc), zeta)  analysis.cpp:71-91,
 *                        scoring.cpp:105-124; glo / loc [units][L] fp32 -> rate [units] fp64
 *                        (device); zeta in (0, 1]; no mass -> EMS_DEGENERATE_INPUT.
 *   ems_redundancy_rate: redundancy_rate_direct(k_raw, v_raw, tau)  analysis.cpp:93-118;
 *                        k / v [units][L][d] (dtype) -> rate [units] fp64 (device). */
EMS_API size_t ems_diagnostics_workspace_bytes(int32_t units, int32_t L);
EMS_API int ems_sparsity_rate(int32_t units, int32_t L, const float* glo, const float* loc, double zeta,
                              double* rate, void* workspace, size_t workspace_bytes, cudaStream_t stream);
EMS_API int ems_redundancy_rate(int32_t dtype, int32_t d, int32_t units, int32_t L, const void* k, const void* v,
                                double tau, double* rate, void* workspace, size_t workspace_bytes,
                                cudaStream_t stream);

/* Synchronises `stream` and returns the first data-dependent error the kernels
 * recorded in the workspace (EMS_DEGENERATE_INPUT, EMS_CORRUPTION) or EMS_OK. */
EMS_API int ems_sync_status(const ems_desc* desc, void* workspace, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* EMS_B200_H */
