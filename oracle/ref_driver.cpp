// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference sources.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with /root/reference/proj/src/*.cpp (in place, read-only) into
// oracle/_ref/libems_ref.so.  It lets the Python tests and bench.py's
// reference arm call the reference's own operator API:
//   prefill_attention      proj/src/scoring.cpp:93-103
//   three_step_scores      proj/src/reference.cpp:51-98
//   init_score_state       proj/src/scoring.cpp:154-162
//   compress_prefill       proj/src/compressor.cpp:163-242
//   cache_dump_json        proj/src/cache.cpp:114-150
//   make_engine / prefill  proj/src/engine.cpp:26-82
//   gen_synthetic          proj/src/trace.cpp:414-429
// No reference code is copied here; everything is a call into it.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "ems/analysis.hpp"
#include "ems/compressor.hpp"
#include "ems/engine.hpp"
#include "ems/errors.hpp"
#include "ems/policies.hpp"
#include "ems/reference.hpp"
#include "ems/scoring.hpp"
#include "ems/trace.hpp"

namespace {

thread_local std::string g_err;
thread_local std::string g_json;

ems::Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
    ems::Matrix m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(double) * rows * cols);
    return m;
}

ems::CompressionConfig make_config(int64_t n_budget, int64_t l_win, double tau, double gamma,
                                   int64_t kernel, int32_t zero_class) {
    ems::CompressionConfig c;
    c.n_budget = static_cast<std::size_t>(n_budget);
    c.l_win = static_cast<std::size_t>(l_win);
    c.tau = tau;
    c.gamma = gamma;
    c.kernel_size = static_cast<std::size_t>(kernel);
    c.eviction = zero_class ? ems::EvictionRealization::zero_class
                            : ems::EvictionRealization::explicit_removal;
    return c;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ems::DegenerateInputError& e) {
        g_err = e.what();
        return 2;
    } catch (const ems::CorruptionError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // namespace

extern "C" {

const char* ems_ref_last_error() { return g_err.c_str(); }
const char* ems_ref_last_json() { return g_json.c_str(); }
int ems_ref_max_threads() { return omp_get_max_threads(); }

int ems_ref_prefill_attention(const double* q, const double* k, const double* v, int64_t n,
                              int64_t d, int64_t l_win, double* out, double* glo, double* loc) {
    return guarded([&] {
        const auto Q = to_matrix(q, n, d), K = to_matrix(k, n, d);
        if (v != nullptr) {
            const auto V = to_matrix(v, n, d);
            const ems::PrefillAttention pa = ems::prefill_attention(Q, K, V, l_win);
            if (out) std::memcpy(out, pa.outputs.data.data(), sizeof(double) * n * d);
            std::memcpy(glo, pa.glo.data(), sizeof(double) * n);
            std::memcpy(loc, pa.loc.data(), sizeof(double) * n);
        } else {
            const ems::PrefillScores ps = ems::prefill_scores(Q, K, l_win);
            std::memcpy(glo, ps.glo.data(), sizeof(double) * n);
            std::memcpy(loc, ps.loc.data(), sizeof(double) * n);
        }
    });
}

int ems_ref_three_step_scores(const double* q, const double* k, int64_t n, int64_t d,
                              int64_t l_win, double* glo, double* loc) {
    return guarded([&] {
        const ems::PrefillScores ps =
            ems::reference::three_step_scores(to_matrix(q, n, d), to_matrix(k, n, d), l_win);
        std::memcpy(glo, ps.glo.data(), sizeof(double) * n);
        std::memcpy(loc, ps.loc.data(), sizeof(double) * n);
    });
}

int ems_ref_effective_score(const double* glo, const double* loc_past, const double* loc_cur,
                            int64_t n, int64_t kernel, double* out) {
    return guarded([&] {
        ems::ScoreState s;
        s.glo.assign(glo, glo + n);
        s.loc_past.assign(loc_past, loc_past + n);
        s.loc_cur.assign(loc_cur, loc_cur + n);
        const ems::Vector p = ems::effective_score(s, kernel);
        std::memcpy(out, p.data(), sizeof(double) * n);
    });
}

int ems_ref_sparsity_rate(const double* score, int64_t n, double zeta, double* rate) {
    return guarded([&] { *rate = ems::sparsity_rate(ems::Vector(score, score + n), zeta); });
}

int ems_ref_redundancy_rate_direct(const double* k, const double* v, int64_t n, int64_t d, double tau,
                                   double* rate) {
    return guarded([&] { *rate = ems::redundancy_rate_direct(to_matrix(k, n, d), to_matrix(v, n, d), tau); });
}

// compress_prefill on one head; the resulting HeadCacheState is returned as
// cache_dump_json text (fetch with ems_ref_last_json).
int ems_ref_compress_prefill(const double* k_raw, const double* v_raw, const double* glo,
                             const double* loc, int64_t n, int64_t d, int64_t n_budget,
                             int64_t l_win, double tau, double gamma, int64_t kernel,
                             int32_t zero_class) {
    return guarded([&] {
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        const ems::ScoreState s = ems::init_score_state(ems::Vector(glo, glo + n),
                                                        ems::Vector(loc, loc + n), l_win);
        const ems::HeadCacheState cache =
            ems::compress_prefill(to_matrix(k_raw, n, d), to_matrix(v_raw, n, d), s, cfg);
        g_json = ems::cache_dump_json(cache);
    });
}

// policy_prefill_compress (proj/src/policies.cpp:131-180) on one head: the reference's
// baseline policies.  policy: 0 ems, 1 full, 2 streaming_llm, 3 h2o, 4 snapkv (the C ABI's
// numbering, not PolicyKind's).
int ems_ref_policy_prefill(int32_t policy, int64_t sink, const double* k_raw, const double* v_raw,
                           const double* glo, const double* loc, int64_t n, int64_t d, int64_t n_budget,
                           int64_t l_win, double tau, double gamma, int64_t kernel, int32_t zero_class) {
    return guarded([&] {
        static const ems::PolicyKind kinds[] = {ems::PolicyKind::ems, ems::PolicyKind::full,
                                                ems::PolicyKind::streaming_llm, ems::PolicyKind::h2o,
                                                ems::PolicyKind::snapkv};
        if (policy < 0 || policy > 4) throw std::invalid_argument("policy code");
        ems::PolicyHandle ph{kinds[policy]};
        ph.sink_count = (std::size_t)sink;
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        const ems::ScoreState s = ems::init_score_state(ems::Vector(glo, glo + n),
                                                        ems::Vector(loc, loc + n), l_win);
        const ems::HeadCacheState cache =
            ems::policy_prefill_compress(ph, to_matrix(k_raw, n, d), to_matrix(v_raw, n, d), s, cfg);
        g_json = ems::cache_dump_json(cache);
    });
}

// engine::prefill then `steps` decode_step calls (EMS policy, proj/src/engine.cpp:42-210):
// q/k/v [H][n][d] raw prompt, dq/dk/dv [steps][H][d] raw decode tokens.  Writes
// out [steps][H][d] and argmax [steps][H]; the json buffer receives, per head, the
// prefill cache dump then the final cache dump, separated by '\x1e'.
int ems_ref_engine_decode(const double* q, const double* k, const double* v, const double* dq,
                          const double* dk, const double* dv, int64_t H, int64_t n, int64_t d,
                          int64_t steps, int64_t n_budget, int64_t l_win, double tau, double gamma,
                          int64_t kernel, int32_t zero_class, int32_t without_pos, double rope_base,
                          double* out, int64_t* argmax, int32_t policy, int64_t sink) {
    return guarded([&] {
        auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        if (without_pos) cfg.position_mode = ems::PositionMode::without_pos;
        static const ems::PolicyKind kinds[] = {ems::PolicyKind::ems, ems::PolicyKind::full,
                                                ems::PolicyKind::streaming_llm, ems::PolicyKind::h2o,
                                                ems::PolicyKind::snapkv};
        ems::PolicyHandle ph{kinds[policy]};
        ph.sink_count = (std::size_t)sink;
        ems::EngineState e = ems::make_engine(H, d, ph, cfg, rope_base);
        std::vector<ems::Matrix> qb, kb, vb;
        for (int64_t h = 0; h < H; ++h) {
            qb.push_back(to_matrix(q + h * n * d, n, d));
            kb.push_back(to_matrix(k + h * n * d, n, d));
            vb.push_back(to_matrix(v + h * n * d, n, d));
        }
        ems::prefill(e, qb, kb, vb);
        std::vector<std::string> pre;
        for (int64_t h = 0; h < H; ++h) pre.push_back(ems::cache_dump_json(e.heads[h]));
        for (int64_t s = 0; s < steps; ++s) {
            std::vector<ems::Vector> qs, ks, vs;
            for (int64_t h = 0; h < H; ++h) {
                const size_t o = (size_t)(s * H + h) * d;
                qs.emplace_back(dq + o, dq + o + d);
                ks.emplace_back(dk + o, dk + o + d);
                vs.emplace_back(dv + o, dv + o + d);
            }
            const ems::DecodeResult r = ems::decode_step(e, qs, ks, vs);
            for (int64_t h = 0; h < H; ++h) {
                std::copy(r.per_head[h].begin(), r.per_head[h].end(), out + (size_t)(s * H + h) * d);
                argmax[s * H + h] = r.argmax_position[h];
            }
        }
        g_json.clear();
        for (int64_t h = 0; h < H; ++h) {
            g_json += pre[h];
            g_json += '\x1e';
            g_json += ems::cache_dump_json(e.heads[h]);
            g_json += '\x1e';
        }
    });
}

// The timed composition of the reference arm for one KV
// unit: per query head prefill_attention in parallel over heads (engine.cpp:65),
// GQA mean (contract D2), init_score_state, compress_prefill.  q_rot [G][n][d].
int ems_ref_prefill_unit(const double* q_rot, const double* k_rot, const double* k_raw,
                         const double* v, int64_t G, int64_t n, int64_t d, int64_t n_budget,
                         int64_t l_win, double tau, double gamma, int64_t kernel,
                         int32_t zero_class, double* glo_out, double* loc_out, int32_t dump) {
    return guarded([&] {
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        const auto K = to_matrix(k_rot, n, d), V = to_matrix(v, n, d);
        const std::size_t l_win_eff = std::min<std::size_t>(l_win, n);
        std::vector<ems::PrefillAttention> pa(G);
        std::vector<std::string> errs(G);
#pragma omp parallel for schedule(static)
        for (int64_t h = 0; h < G; ++h) {
            try {
                pa[h] = ems::prefill_attention(to_matrix(q_rot + h * n * d, n, d), K, V, l_win_eff);
            } catch (const std::exception& e) {
                errs[h] = e.what();
            }
        }
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
        ems::Vector glo(n, 0.0), loc(n, 0.0);
        for (int64_t h = 0; h < G; ++h)
            for (int64_t j = 0; j < n; ++j) glo[j] += pa[h].glo[j], loc[j] += pa[h].loc[j];
        for (int64_t j = 0; j < n; ++j) glo[j] /= double(G), loc[j] /= double(G);
        if (glo_out) std::memcpy(glo_out, glo.data(), sizeof(double) * n);
        if (loc_out) std::memcpy(loc_out, loc.data(), sizeof(double) * n);
        const ems::ScoreState s = ems::init_score_state(glo, loc, l_win);
        const ems::HeadCacheState cache = ems::policy_prefill_compress(
            ems::PolicyHandle{ems::PolicyKind::ems}, to_matrix(k_raw, n, d), V, s, cfg);
        if (dump) g_json = ems::cache_dump_json(cache);
    });
}

// The same composition over U units at once, the way engine::prefill spreads work
// (engine.cpp:65: one parallel loop over every head): the U*G (unit, query head) score passes
// share one OpenMP region; when there are fewer of them than threads, each takes
// threads / (U*G) threads for streaming_pass's own row loop (scoring.cpp:41, nested).  Then
// GQA mean, init_score_state and policy_prefill_compress per unit, parallel over units.
//   q_rot [U][G][n][d], k_rot / k_raw / v [U][n][d]; glo_out / loc_out [U][n] (may be NULL).
//   with_out = 1: prefill_attention (O computed and discarded, as engine::prefill's result);
//   0: prefill_scores (same glo/loc, scoring.hpp:48-54).  dump = 1: the caches'
//   cache_dump_json texts, '\x1e'-terminated in unit order (ems_ref_last_json).
//   seconds (may be NULL) <- {score passes, GQA mean + compress} wall time (omp_get_wtime).
int ems_ref_prefill_units(const double* q_rot, const double* k_rot, const double* k_raw, const double* v,
                          int64_t U, int64_t G, int64_t n, int64_t d, int64_t n_budget, int64_t l_win,
                          double tau, double gamma, int64_t kernel, int32_t zero_class, int32_t with_out,
                          double* glo_out, double* loc_out, int32_t dump, double* seconds) {
    return guarded([&] {
        const double t0 = omp_get_wtime();
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        const std::size_t l_win_eff = std::min<std::size_t>(l_win, n);
        const int64_t items = U * G;
        const int T = omp_get_max_threads();
        const int outer = (int)std::min<int64_t>(items, T);
        const int inner = std::max(1, T / std::max(outer, 1));
        const int levels = omp_get_max_active_levels();
        omp_set_max_active_levels(inner > 1 ? 2 : 1);
        std::vector<ems::Vector> glo(items), loc(items);
        std::vector<std::string> errs(items);
#pragma omp parallel for num_threads(outer) schedule(dynamic, 1)
        for (int64_t it = 0; it < items; ++it) {
            omp_set_num_threads(inner);
            const int64_t u = it / G;
            try {
                const auto Q = to_matrix(q_rot + it * n * d, n, d), K = to_matrix(k_rot + u * n * d, n, d);
                if (with_out) {
                    ems::PrefillAttention pa =
                        ems::prefill_attention(Q, K, to_matrix(v + u * n * d, n, d), l_win_eff);
                    glo[it] = std::move(pa.glo);
                    loc[it] = std::move(pa.loc);
                } else {
                    ems::PrefillScores ps = ems::prefill_scores(Q, K, l_win_eff);
                    glo[it] = std::move(ps.glo);
                    loc[it] = std::move(ps.loc);
                }
            } catch (const std::exception& e) {
                errs[it] = e.what();
            }
        }
        omp_set_max_active_levels(levels);
        for (auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
        const double t1 = omp_get_wtime();
        std::vector<std::string> dumps(U);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t u = 0; u < U; ++u) {
            ems::Vector g(n, 0.0), l(n, 0.0);
            for (int64_t h = 0; h < G; ++h)
                for (int64_t j = 0; j < n; ++j) g[j] += glo[u * G + h][j], l[j] += loc[u * G + h][j];
            for (int64_t j = 0; j < n; ++j) g[j] /= double(G), l[j] /= double(G);
            if (glo_out) std::memcpy(glo_out + u * n, g.data(), sizeof(double) * n);
            if (loc_out) std::memcpy(loc_out + u * n, l.data(), sizeof(double) * n);
            try {
                const ems::ScoreState s = ems::init_score_state(g, l, l_win);
                const ems::HeadCacheState cache =
                    ems::policy_prefill_compress(ems::PolicyHandle{ems::PolicyKind::ems},
                                                 to_matrix(k_raw + u * n * d, n, d),
                                                 to_matrix(v + u * n * d, n, d), s, cfg);
                if (dump) dumps[u] = ems::cache_dump_json(cache);
            } catch (const std::exception& e) {
                dumps[u] = std::string("\x1f") + e.what();
            }
        }
        if (seconds) {
            seconds[0] = t1 - t0;
            seconds[1] = omp_get_wtime() - t1;
        }
        g_json.clear();
        for (auto& s : dumps) {
            if (!s.empty() && s[0] == '\x1f') throw std::invalid_argument(s.substr(1));
            g_json += s;
            g_json += '\x1e';
        }
    });
}

// engine::prefill with the EMS policy over raw per-head blocks [H][n][d]
// (RoPE applied inside, engine.cpp:68-69); dumps head `dump_head`'s cache.
int ems_ref_engine_prefill(const double* q, const double* k, const double* v, int64_t H,
                           int64_t n, int64_t d, int64_t n_budget, int64_t l_win, double tau,
                           double gamma, int64_t kernel, int32_t zero_class, double rope_base,
                           int64_t dump_head) {
    return guarded([&] {
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        ems::EngineState e =
            ems::make_engine(H, d, ems::PolicyHandle{ems::PolicyKind::ems}, cfg, rope_base);
        std::vector<ems::Matrix> qb, kb, vb;
        for (int64_t h = 0; h < H; ++h) {
            qb.push_back(to_matrix(q + h * n * d, n, d));
            kb.push_back(to_matrix(k + h * n * d, n, d));
            vb.push_back(to_matrix(v + h * n * d, n, d));
        }
        ems::prefill(e, qb, kb, vb);
        g_json = ems::cache_dump_json(e.heads[dump_head]);
    });
}

// ---- the fine-grained operators, for the C++ API test (tests/cpp/test_ems_hpp.cpp) ----------
// partition_tokens (compressor.cpp:48-74) -> class bytes: 0 irrelevant, 1 TBM, 2 important, 3 local.
int ems_ref_partition_tokens(const double* pooled, int64_t n, int64_t n_budget, int64_t l_win, double gamma,
                             int8_t* cls) {
    return guarded([&] {
        const auto cfg = make_config(n_budget, l_win, 0.6, gamma, 1, 1);
        const ems::TokenPartition p = ems::partition_tokens(ems::Vector(pooled, pooled + n), cfg);
        for (auto i : p.irrelevant) cls[i] = 0;
        for (auto i : p.tbm) cls[i] = 1;
        for (auto i : p.important) cls[i] = 2;
        for (auto i : p.local) cls[i] = 3;
    });
}

// assign_merge_destinations (compressor.cpp:76-95).
int ems_ref_assign_merge_destinations(const double* r, int64_t rows, int64_t cols, double tau, int32_t* dest) {
    return guarded([&] {
        const auto d = ems::assign_merge_destinations(to_matrix(r, rows, cols), tau);
        std::copy(d.begin(), d.end(), dest);
    });
}

// weighted_merge (compressor.cpp:97-161) on a cache whose slot c holds center column c; writes the
// merged centers back and the appended LUT entries (lut_pos / lut_slot, *n_lut of them).
int ems_ref_weighted_merge(int64_t d, int64_t n_cols, double* center_unit_key, double* center_value,
                           double* center_score, const double* center_weight, int64_t n_tbm, const double* tbm_k,
                           const double* tbm_v, const int64_t* tbm_pos, const double* tbm_w, const double* tbm_score,
                           const int32_t* dest, int32_t zero_class, int64_t* lut_pos, int32_t* lut_slot,
                           int64_t* n_lut) {
    return guarded([&] {
        ems::HeadCacheState cache;
        cache.head_dim = (std::size_t)d;
        std::vector<std::int32_t> slot_by_col(n_cols);
        for (int64_t c = 0; c < n_cols; ++c) {
            ems::CenterEntry e;
            e.unit_key.assign(center_unit_key + c * d, center_unit_key + (c + 1) * d);
            e.value.assign(center_value + c * d, center_value + (c + 1) * d);
            e.score = ems::ScoreTriple{center_score[3 * c], center_score[3 * c + 1], center_score[3 * c + 2]};
            slot_by_col[c] = cache.insert_center(std::move(e));
        }
        ems::TbmTokens t;
        t.k_raw = to_matrix(tbm_k, n_tbm, d);
        t.v_raw = to_matrix(tbm_v, n_tbm, d);
        t.positions.assign(tbm_pos, tbm_pos + n_tbm);
        t.weights.assign(tbm_w, tbm_w + n_tbm);
        for (int64_t i = 0; i < n_tbm; ++i)
            t.score_triples.push_back(ems::ScoreTriple{tbm_score[3 * i], tbm_score[3 * i + 1], tbm_score[3 * i + 2]});
        const auto cfg = make_config(64, 8, 0.6, 4.0, 1, zero_class);
        ems::weighted_merge(cache, slot_by_col, ems::Vector(center_weight, center_weight + n_cols), t,
                            std::vector<std::int32_t>(dest, dest + n_tbm), cfg);
        for (int64_t c = 0; c < n_cols; ++c) {
            const ems::CenterEntry& e = *cache.slots[slot_by_col[c]];
            std::copy(e.unit_key.begin(), e.unit_key.end(), center_unit_key + c * d);
            std::copy(e.value.begin(), e.value.end(), center_value + c * d);
            center_score[3 * c] = e.score.glo, center_score[3 * c + 1] = e.score.loc_past,
                         center_score[3 * c + 2] = e.score.loc_cur;
        }
        *n_lut = (int64_t)cache.lut.size();
        for (std::size_t i = 0; i < cache.lut.size(); ++i) lut_pos[i] = cache.lut[i].position, lut_slot[i] = cache.lut[i].slot;
    });
}

// engine::prefill (make_engine + prefill, engine.cpp:26-82) over raw blocks [H][n][d] with any
// policy (0 ems, 1 full, 2 streaming_llm, 3 h2o, 4 snapkv): outputs [H][n][d]; per head the center
// positions (slot order, [H][cap_c], n_centers [H]), the LUT ([H][cap_lut], n_lut [H]) and the
// compressed flag.
int ems_ref_engine_prefill_arrays(const double* q, const double* k, const double* v, int64_t H, int64_t n, int64_t d,
                                  int64_t n_budget, int64_t l_win, double tau, double gamma, int64_t kernel,
                                  int32_t zero_class, double rope_base, int32_t policy, int64_t sink, double* out,
                                  int64_t cap_c, int64_t* center_pos, int64_t* n_centers, int64_t cap_lut,
                                  int64_t* lut_pos, int32_t* lut_slot, int64_t* n_lut, int32_t* compressed) {
    return guarded([&] {
        static const ems::PolicyKind kinds[] = {ems::PolicyKind::ems, ems::PolicyKind::full,
                                                ems::PolicyKind::streaming_llm, ems::PolicyKind::h2o,
                                                ems::PolicyKind::snapkv};
        ems::PolicyHandle ph{kinds[policy]};
        ph.sink_count = (std::size_t)sink;
        const auto cfg = make_config(n_budget, l_win, tau, gamma, kernel, zero_class);
        ems::EngineState e = ems::make_engine(H, d, ph, cfg, rope_base);
        std::vector<ems::Matrix> qb, kb, vb;
        for (int64_t h = 0; h < H; ++h) {
            qb.push_back(to_matrix(q + h * n * d, n, d));
            kb.push_back(to_matrix(k + h * n * d, n, d));
            vb.push_back(to_matrix(v + h * n * d, n, d));
        }
        const ems::PrefillResult r = ems::prefill(e, qb, kb, vb);
        for (int64_t h = 0; h < H; ++h) {
            std::memcpy(out + h * n * d, r.per_head[h].outputs.data.data(), sizeof(double) * n * d);
            const ems::HeadCacheState& c = e.heads[h];
            int64_t nc = 0;
            for (const auto& s : c.slots)
                if (s.has_value() && nc < cap_c) center_pos[h * cap_c + nc++] = s->position;
            n_centers[h] = nc;
            n_lut[h] = std::min<int64_t>((int64_t)c.lut.size(), cap_lut);
            for (int64_t i = 0; i < n_lut[h]; ++i)
                lut_pos[h * cap_lut + i] = c.lut[i].position, lut_slot[h * cap_lut + i] = c.lut[i].slot;
            compressed[h] = c.compressed;
        }
    });
}

// gen_synthetic prefill step, blocks laid out [H][n][d] (fp64 holding f32 values).
int ems_ref_gen_synthetic(int32_t kind, uint64_t seed, int64_t tokens, int64_t heads, int64_t dim,
                          int64_t decode_steps, double level, double perturb, double* q, double* k,
                          double* v) {
    return guarded([&] {
        ems::SynthParams p;
        p.tokens = tokens;
        p.heads = heads;
        p.dim = dim;
        p.decode_steps = decode_steps;
        p.level = level;
        p.perturb = perturb;
        const ems::Trace t = ems::gen_synthetic(static_cast<ems::SynthKind>(kind), seed, p);
        const ems::TraceStep& s = t.steps.at(0);
        for (int64_t h = 0; h < heads; ++h) {
            std::memcpy(q + h * tokens * dim, s.q[h].data.data(), sizeof(double) * tokens * dim);
            std::memcpy(k + h * tokens * dim, s.k[h].data.data(), sizeof(double) * tokens * dim);
            std::memcpy(v + h * tokens * dim, s.v[h].data.data(), sizeof(double) * tokens * dim);
        }
    });
}

// gen_synthetic + save_trace (proj/src/trace.cpp:157-179): a reference-written KVTR file.
int ems_ref_save_synthetic(int32_t kind, uint64_t seed, int64_t tokens, int64_t heads, int64_t dim,
                           int64_t decode_steps, double level, double depth, const char* path) {
    return guarded([&] {
        ems::SynthParams p;
        p.tokens = tokens;
        p.heads = heads;
        p.dim = dim;
        p.decode_steps = decode_steps;
        p.level = level;
        p.depth = depth;
        ems::save_trace(ems::gen_synthetic(static_cast<ems::SynthKind>(kind), seed, p), path);
    });
}

// load_trace (proj/src/trace.cpp:119-155): 0 if the reference reader accepts the file, else the
// FormatError offset is written to *offset and 3 returned.
int ems_ref_load_trace(const char* path, int64_t* offset) {
    try {
        ems::load_trace(path);
        return 0;
    } catch (const ems::FormatError& e) {
        *offset = (int64_t)e.offset;
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// gen_synthetic (proj/src/trace.cpp:239-410) with every step: q/k/v [heads][tokens + steps][dim],
// prompt rows first, then one row per decode step.  depth: needle position fraction.
int ems_ref_gen_trace(int32_t kind, uint64_t seed, int64_t tokens, int64_t heads, int64_t dim,
                      int64_t decode_steps, double level, double depth, double* q, double* k, double* v) {
    return guarded([&] {
        ems::SynthParams p;
        p.tokens = tokens;
        p.heads = heads;
        p.dim = dim;
        p.decode_steps = decode_steps;
        p.level = level;
        p.depth = depth;
        const ems::Trace t = ems::gen_synthetic(static_cast<ems::SynthKind>(kind), seed, p);
        const int64_t T = tokens + decode_steps;
        for (int64_t h = 0; h < heads; ++h) {
            const ems::TraceStep& s0 = t.steps.at(0);
            std::memcpy(q + h * T * dim, s0.q[h].data.data(), sizeof(double) * tokens * dim);
            std::memcpy(k + h * T * dim, s0.k[h].data.data(), sizeof(double) * tokens * dim);
            std::memcpy(v + h * T * dim, s0.v[h].data.data(), sizeof(double) * tokens * dim);
            for (int64_t s = 0; s < decode_steps; ++s) {
                const ems::TraceStep& st = t.steps.at(1 + s);
                const size_t o = (size_t)(h * T + tokens + s) * dim;
                std::memcpy(q + o, st.q[h].data.data(), sizeof(double) * dim);
                std::memcpy(k + o, st.k[h].data.data(), sizeof(double) * dim);
                std::memcpy(v + o, st.v[h].data.data(), sizeof(double) * dim);
            }
        }
    });
}

}  // extern "C"
