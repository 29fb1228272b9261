// ems_b200/ems.hpp -- the reference's C++ operator API, restored on top of the C ABI.
//
// Drop-in for the prefill path of the EMS reference (proj/include/ems/*.hpp): the
// same type names, entry-point names, argument order and meaning, and the same
// exception types, in namespace ems_b200.  A reference caller switches with
//     namespace ems = ems_b200;   // or: using ems_b200::prefill_attention; ...
// Inputs are host fp64 `Matrix` objects exactly as in the reference
// (proj/include/ems/types.hpp:13-34); they are rounded once to the device dtype
// (fp32 by default, bf16 on request), run through the sm_100a kernels of
// libems_b200.so, and the results come back as fp64 host objects.  The batched,
// zero-copy device API is the C ABI in ems_b200.h; this header is the
// reference-shaped convenience layer (one host<->device round trip per call).
//
// Link: -lems_b200 -lcudart  (header-only otherwise).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ems_b200.h"

namespace ems_b200 {

// ---------------------------------------------------------------- types (types.hpp, cache.hpp)
using Vector = std::vector<double>;

struct Matrix {  // proj/include/ems/types.hpp:13-34
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    double at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    Vector row_vec(std::size_t r) const {
        return Vector(data.begin() + r * cols, data.begin() + (r + 1) * cols);
    }
};

enum class EvictionRealization { zero_class, explicit_removal };

struct CompressionConfig {  // proj/include/ems/cache.hpp:20-39
    std::size_t n_budget = 256;
    std::size_t l_win = 32;
    double tau = 0.6;
    double gamma = 4.0;
    double zeta = 0.95;
    std::size_t kernel_size = 7;
    EvictionRealization eviction = EvictionRealization::zero_class;
    bool key_only_similarity = false;  // contract D1 flag (reference: cos_k * cos_v)
    std::size_t center_capacity() const { return n_budget - l_win; }
    std::size_t tbm_target() const { return static_cast<std::size_t>((gamma - 1.0) * double(n_budget)); }
    std::size_t lut_capacity() const { return static_cast<std::size_t>(gamma * double(n_budget)); }
};

struct ScoreTriple {
    double glo = 0.0, loc_past = 0.0, loc_cur = 0.0;
};
struct CenterEntry {
    Vector unit_key;
    double key_norm = 0.0;
    Vector value;
    std::int64_t position = 0;
    ScoreTriple score;
};
struct LocalEntry {
    Vector key, value;
    std::int64_t position = 0;
    ScoreTriple score;
};
inline constexpr std::int32_t kZeroClass = -1;
struct LutEntry {
    std::int64_t position = 0;
    std::int32_t slot = kZeroClass;
};
struct HeadCacheState {  // proj/include/ems/cache.hpp:81-111 (prefill subset)
    std::size_t head_dim = 0;
    std::vector<std::optional<CenterEntry>> slots;
    std::deque<LocalEntry> locals;
    std::vector<LutEntry> lut;
    bool compressed = false;
};
struct ScoreState {  // proj/include/ems/scoring.hpp:13-24
    Vector glo, loc_past, loc_cur;
    std::size_t window_fill = 0;
    std::size_t l_win = 0;
    std::size_t size() const { return glo.size(); }
};
struct PrefillScores {
    Vector glo, loc;
};
struct PrefillAttention {
    Matrix outputs;
    Vector glo, loc;
};
struct TokenPartition {  // proj/include/ems/compressor.hpp:14-20
    std::vector<std::size_t> irrelevant, tbm, important, local;
};

// ---------------------------------------------------------------- errors (errors.hpp)
class DegenerateInputError : public std::runtime_error {
   public:
    explicit DegenerateInputError(const std::string& w) : std::runtime_error(w) {}
};
class CorruptionError : public std::runtime_error {
   public:
    explicit CorruptionError(const std::string& w) : std::runtime_error(w) {}
};
class CudaError : public std::runtime_error {
   public:
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {

inline void check(int status) {
    if (status == EMS_OK) return;
    const std::string msg = ems_last_error();
    switch (status) {
        case EMS_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EMS_DEGENERATE_INPUT: throw DegenerateInputError(msg);
        case EMS_CORRUPTION: throw CorruptionError(msg);
        default: throw CudaError(msg);
    }
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
}

// RAII device buffer.
struct DevBuf {
    void* p = nullptr;
    std::size_t n = 0;
    explicit DevBuf(std::size_t bytes) : n(bytes) {
        if (bytes) cuda(cudaMalloc(&p, bytes));
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Host fp64 -> device dtype (one rounding), laid out contiguously.
inline DevBuf upload(const std::vector<const Matrix*>& ms, int dtype) {
    std::size_t total = 0;
    for (auto* m : ms) total += m->data.size();
    const std::size_t es = dtype == EMS_F32 ? 4 : 2;
    DevBuf d(total * es);
    std::vector<unsigned char> h(total * es);
    std::size_t o = 0;
    for (auto* m : ms)
        for (double x : m->data) {
            if (dtype == EMS_F32) {
                const float f = static_cast<float>(x);
                std::memcpy(&h[o * 4], &f, 4);
            } else {
                const __nv_bfloat16 b = __float2bfloat16_rn(static_cast<float>(x));
                std::memcpy(&h[o * 2], &b, 2);
            }
            ++o;
        }
    cuda(cudaMemcpy(d.p, h.data(), h.size(), cudaMemcpyHostToDevice));
    return d;
}

inline std::vector<double> download(const void* dev, std::size_t n, int dtype) {
    const std::size_t es = dtype == EMS_F32 ? 4 : 2;
    std::vector<unsigned char> h(n * es);
    cuda(cudaMemcpy(h.data(), dev, h.size(), cudaMemcpyDeviceToHost));
    std::vector<double> out(n);
    for (std::size_t i = 0; i < n; ++i) {
        if (dtype == EMS_F32) {
            float f;
            std::memcpy(&f, &h[i * 4], 4);
            out[i] = f;
        } else {
            __nv_bfloat16 b;
            std::memcpy(&b, &h[i * 2], 2);
            out[i] = __bfloat162float(b);
        }
    }
    return out;
}

template <class T>
std::vector<T> download_raw(const void* dev, std::size_t n) {
    std::vector<T> out(n);
    cuda(cudaMemcpy(out.data(), dev, n * sizeof(T), cudaMemcpyDeviceToHost));
    return out;
}

inline ems_desc make_desc(std::size_t heads_q, std::size_t heads_kv, std::size_t n, std::size_t d,
                          int dtype, const CompressionConfig& c) {
    ems_desc desc{};
    desc.batch = 1;
    desc.heads_q = static_cast<int32_t>(heads_q);
    desc.heads_kv = static_cast<int32_t>(heads_kv);
    desc.seq_len = static_cast<int32_t>(n);
    desc.head_dim = static_cast<int32_t>(d);
    desc.dtype = dtype;
    desc.l_win = static_cast<int32_t>(c.l_win);
    desc.n_budget = static_cast<int32_t>(c.n_budget);
    desc.tau = c.tau;
    desc.gamma = c.gamma;
    desc.kernel_size = static_cast<int32_t>(c.kernel_size);
    desc.zero_class = c.eviction == EvictionRealization::zero_class;
    desc.key_only = c.key_only_similarity;
    desc.score_impl = EMS_SCORE_AUTO;
    desc.first_position = 0;
    return desc;
}

// Score pass on one group of G query heads sharing one KV head.
inline void score_group(const std::vector<const Matrix*>& q, const Matrix& k, const Matrix* v,
                        std::size_t l_win, int dtype, std::vector<Matrix>* outs, Vector& glo,
                        Vector& loc) {
    const std::size_t n = k.rows, d = k.cols, G = q.size();
    for (auto* m : q)
        if (m->rows != n || m->cols != d)
            throw std::invalid_argument("prefill scores: Q/K shape mismatch");  // scoring.cpp:22-24
    if (n == 0) throw std::invalid_argument("prefill scores: empty block");
    if (v && v->rows != n) throw std::invalid_argument("prefill_attention: V token count mismatch");
    CompressionConfig c;
    c.l_win = std::max<std::size_t>(l_win, 1);
    c.n_budget = c.l_win + 1;
    c.gamma = 1.0;
    c.kernel_size = 1;
    ems_desc desc = make_desc(G, 1, n, d, dtype, c);
    DevBuf dq = upload(q, dtype), dk = upload({&k}, dtype);
    DevBuf dv = v ? upload({v}, dtype) : DevBuf(0);
    const std::size_t es = dtype == EMS_F32 ? 4 : 2;
    DevBuf dout(outs ? G * n * d * es : 0);
    DevBuf dglo(n * 4), dloc(n * 4);
    DevBuf ws(ems_workspace_bytes(&desc));
    check(ems_score(&desc, dq.p, dk.p, v ? dv.p : nullptr, outs ? dout.p : nullptr, nullptr,
                    dglo.as<float>(), dloc.as<float>(), ws.p, ws.n, nullptr));
    cuda(cudaDeviceSynchronize());
    const auto g = download_raw<float>(dglo.p, n), l = download_raw<float>(dloc.p, n);
    glo.assign(g.begin(), g.end());
    loc.assign(l.begin(), l.end());
    if (outs) {
        const auto o = download(dout.p, G * n * d, dtype);
        outs->assign(G, Matrix(n, d));
        for (std::size_t h = 0; h < G; ++h)
            std::copy(o.begin() + h * n * d, o.begin() + (h + 1) * n * d, (*outs)[h].data.begin());
    }
}

}  // namespace detail

// ---------------------------------------------------------------- scoring.hpp
// tile_rows is accepted for signature compatibility; results do not depend on it
// (the reference guarantees the same, test_scoring.cpp:125-136).
inline PrefillScores prefill_scores(const Matrix& q_block, const Matrix& k_block, std::size_t l_win,
                                    std::size_t /*tile_rows*/ = 128, int dtype = EMS_F32) {
    PrefillScores s;
    detail::score_group({&q_block}, k_block, nullptr, std::min(l_win, q_block.rows), dtype, nullptr,
                        s.glo, s.loc);
    return s;
}
inline Vector global_score_prefill(const Matrix& q, const Matrix& k, std::size_t tile_rows = 128) {
    if (q.rows != k.rows || q.cols != k.cols)
        throw std::invalid_argument("prefill scores: Q/K shape mismatch");
    return prefill_scores(q, k, 1, tile_rows).glo;
}
inline Vector local_score_prefill(const Matrix& q, const Matrix& k, std::size_t l_win,
                                  std::size_t tile_rows = 128) {
    if (l_win == 0 || l_win > q.rows)  // scoring.cpp:77-79
        throw std::invalid_argument("local_score_prefill: l_win must be in [1, N]");
    return prefill_scores(q, k, l_win, tile_rows).loc;
}
inline PrefillAttention prefill_attention(const Matrix& q_block, const Matrix& k_block,
                                          const Matrix& v_block, std::size_t l_win,
                                          std::size_t /*tile_rows*/ = 128, int dtype = EMS_F32) {
    PrefillAttention pa;
    std::vector<Matrix> outs;
    detail::score_group({&q_block}, k_block, &v_block, std::min(l_win, q_block.rows), dtype, &outs,
                        pa.glo, pa.loc);
    pa.outputs = std::move(outs[0]);
    return pa;
}

inline Vector combine_glo_loc(const Vector& s_glo, const Vector& s_loc) {  // scoring.cpp:105-124
    if (s_glo.size() != s_loc.size()) throw std::invalid_argument("combine_glo_loc: length mismatch");
    double sg = 0.0, sl = 0.0;
    for (std::size_t i = 0; i < s_glo.size(); ++i) sg += s_glo[i], sl += s_loc[i];
    if (sg <= 0.0) throw DegenerateInputError("combine_glo_loc: global score has no mass");
    Vector out(s_glo.size());
    for (std::size_t i = 0; i < s_glo.size(); ++i) out[i] = std::max(s_glo[i] * (sl / sg), s_loc[i]);
    return out;
}
inline ScoreState init_score_state(Vector glo, Vector loc, std::size_t l_win) {  // scoring.cpp:154-162
    ScoreState s;
    s.glo = std::move(glo);
    s.loc_past = std::move(loc);
    s.loc_cur.assign(s.glo.size(), 0.0);
    s.l_win = l_win;
    return s;
}

// ---------------------------------------------------------------- compressor.hpp / engine
namespace detail {

struct CompressResult {
    HeadCacheState cache;
    std::vector<float> pooled;
    std::vector<int8_t> cls;
};

// compress_prefill on device for one KV head with externally supplied scores.
inline CompressResult compress_device(const Matrix& k_raw, const Matrix& v_raw, const Vector& glo,
                                      const Vector& loc, const CompressionConfig& c, int dtype,
                                      int policy = EMS_POLICY_EMS, std::size_t sink_count = 4) {
    const std::size_t n = k_raw.rows, d = k_raw.cols;
    if (n == 0 || v_raw.rows != n || glo.size() != n || loc.size() != n)
        throw std::invalid_argument("compress_prefill: inconsistent token counts");
    ems_desc desc = make_desc(1, 1, n, d, dtype, c);
    desc.policy = policy;
    desc.sink_count = static_cast<int32_t>(sink_count);
    check(ems_validate(&desc));
    ems_cache_dims dims{};
    check(ems_cache_dims_for(&desc, &dims));
    const std::size_t es = dtype == EMS_F32 ? 4 : 2;
    DevBuf dk = upload({&k_raw}, dtype), dv = upload({&v_raw}, dtype);
    std::vector<float> g(glo.begin(), glo.end()), l(loc.begin(), loc.end());
    DevBuf dg(n * 4), dl(n * 4);
    cuda(cudaMemcpy(dg.p, g.data(), n * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dl.p, l.data(), n * 4, cudaMemcpyHostToDevice));
    const std::size_t C = dims.centers, Lc = dims.locals, U = std::max(dims.lut, 1), T = std::max(dims.tbm, 1);
    DevBuf ck(C * d * es), cn(C * 4), cv(C * d * es), cp(C * 4), cs(C * 12), lk(Lc * d * es),
        lv(Lc * d * es), lp(Lc * 4), ls(Lc * 12), up(U * 4), us(U * 4), cnt(16);
    DevBuf pooled(n * 4), cls(n), imp(C * 4), tbm(T * 4), pc(16), dest(T * 4);
    ems_cache cache{ck.p, cn.as<float>(), cv.p, cp.as<int32_t>(), cs.as<float>(), lk.p, lv.p,
                    lp.as<int32_t>(), ls.as<float>(), up.as<int32_t>(), us.as<int32_t>(), cnt.as<int32_t>()};
    ems_stage stage{pooled.as<float>(), cls.as<int8_t>(), imp.as<int32_t>(), tbm.as<int32_t>(),
                    pc.as<int32_t>(), dest.as<int32_t>()};
    DevBuf ws(ems_workspace_bytes(&desc));
    if (n > c.n_budget && policy != EMS_POLICY_FULL) {
        check(ems_select(&desc, dg.as<float>(), dl.as<float>(), &stage, ws.p, ws.n, nullptr));
        check(ems_merge(&desc, dk.p, dv.p, &stage, ws.p, ws.n, nullptr));
    }
    check(ems_compact(&desc, dk.p, dv.p, dg.as<float>(), dl.as<float>(), &stage, &cache, ws.p, ws.n, nullptr));
    check(ems_sync_status(&desc, ws.p, nullptr));
    const auto counts = download_raw<int32_t>(cnt.p, 4);
    CompressResult r;
    HeadCacheState& hc = r.cache;
    hc.head_dim = d;
    hc.compressed = counts[3] != 0;
    const auto ckh = download(ck.p, C * d, dtype), cvh = download(cv.p, C * d, dtype);
    const auto cnh = download_raw<float>(cn.p, C), csh = download_raw<float>(cs.p, C * 3);
    const auto cph = download_raw<int32_t>(cp.p, C);
    for (int s = 0; s < counts[0]; ++s) {
        CenterEntry e;
        e.unit_key.assign(ckh.begin() + s * d, ckh.begin() + (s + 1) * d);
        e.value.assign(cvh.begin() + s * d, cvh.begin() + (s + 1) * d);
        e.key_norm = cnh[s];
        e.position = cph[s];
        e.score = {csh[3 * s], csh[3 * s + 1], csh[3 * s + 2]};
        hc.slots.emplace_back(std::move(e));
    }
    const auto lkh = download(lk.p, Lc * d, dtype), lvh = download(lv.p, Lc * d, dtype);
    const auto lph = download_raw<int32_t>(lp.p, Lc);
    const auto lsh = download_raw<float>(ls.p, Lc * 3);
    for (int i = 0; i < counts[1]; ++i) {
        LocalEntry e;
        e.key.assign(lkh.begin() + i * d, lkh.begin() + (i + 1) * d);
        e.value.assign(lvh.begin() + i * d, lvh.begin() + (i + 1) * d);
        e.position = lph[i];
        e.score = {lsh[3 * i], lsh[3 * i + 1], lsh[3 * i + 2]};
        hc.locals.push_back(std::move(e));
    }
    const auto uph = download_raw<int32_t>(up.p, U), ush = download_raw<int32_t>(us.p, U);
    for (int i = 0; i < counts[2]; ++i) hc.lut.push_back({uph[i], ush[i]});
    if (n > c.n_budget && policy != EMS_POLICY_FULL) {
        r.pooled = download_raw<float>(pooled.p, n);
        r.cls = download_raw<int8_t>(cls.p, n);
    }
    return r;
}

}  // namespace detail

// compress_prefill, proj/include/ems/compressor.hpp:58-60 (first_position = 0).
inline HeadCacheState compress_prefill(const Matrix& k_raw, const Matrix& v_raw,
                                       const ScoreState& scores, const CompressionConfig& config,
                                       int dtype = EMS_F32) {
    Vector loc(scores.size());
    for (std::size_t i = 0; i < loc.size(); ++i)
        loc[i] = scores.loc_past[i] + (scores.loc_cur.empty() ? 0.0 : scores.loc_cur[i]);
    return detail::compress_device(k_raw, v_raw, scores.glo, loc, config, dtype).cache;
}

// policies.hpp: PolicyKind / PolicyHandle (proj/include/ems/policies.hpp:12-20) and
// policy_prefill_compress (proj/src/policies.cpp:131-180) on the device select/compact kernels.
enum class PolicyKind { full, streaming_llm, h2o, snapkv, ems };
struct PolicyHandle {
    PolicyKind kind = PolicyKind::full;
    std::size_t sink_count = 4;  // streaming_llm
    void validate(const CompressionConfig& config) const {  // policies.cpp:111-116
        if (kind == PolicyKind::streaming_llm && config.n_budget < sink_count + config.l_win)
            throw std::invalid_argument("streaming_llm: n_budget must cover sinks plus the local window");
    }
};
inline int policy_code(PolicyKind k) {
    switch (k) {
        case PolicyKind::full: return EMS_POLICY_FULL;
        case PolicyKind::streaming_llm: return EMS_POLICY_STREAMING;
        case PolicyKind::h2o: return EMS_POLICY_H2O;
        case PolicyKind::snapkv: return EMS_POLICY_SNAPKV;
        case PolicyKind::ems: return EMS_POLICY_EMS;
    }
    return EMS_POLICY_EMS;
}
inline HeadCacheState policy_prefill_compress(const PolicyHandle& policy, const Matrix& k_raw,
                                              const Matrix& v_raw, const ScoreState& scores,
                                              const CompressionConfig& config, int dtype = EMS_F32) {
    policy.validate(config);
    Vector loc(scores.size());
    for (std::size_t i = 0; i < loc.size(); ++i)
        loc[i] = scores.loc_past[i] + (scores.loc_cur.empty() ? 0.0 : scores.loc_cur[i]);
    return detail::compress_device(k_raw, v_raw, scores.glo, loc, config, dtype, policy_code(policy.kind),
                                   policy.sink_count)
        .cache;
}

// partition_tokens on the effective score of a ScoreState (the device select kernel
// computes effective_score itself; the reference takes the pooled vector).
inline TokenPartition partition_tokens_from_scores(const Matrix& k_raw, const Matrix& v_raw,
                                                   const ScoreState& scores,
                                                   const CompressionConfig& config) {
    Vector loc(scores.size());
    for (std::size_t i = 0; i < loc.size(); ++i) loc[i] = scores.loc_past[i];
    const auto r = detail::compress_device(k_raw, v_raw, scores.glo, loc, config, EMS_F32);
    TokenPartition p;
    for (std::size_t i = 0; i < r.cls.size(); ++i) {
        if (r.cls[i] == 2) p.important.push_back(i);
        else if (r.cls[i] == 1) p.tbm.push_back(i);
        else if (r.cls[i] == 0) p.irrelevant.push_back(i);
        else p.local.push_back(i);
    }
    return p;
}

// redundancy_cross, proj/include/ems/analysis.hpp:19-20.
inline Matrix redundancy_cross(const Matrix& k_rows, const Matrix& v_rows, const Matrix& k_cols,
                               const Matrix& v_cols, bool key_only = false) {
    if (k_rows.rows != v_rows.rows || k_cols.rows != v_cols.rows)
        throw std::invalid_argument("redundancy_cross: K/V token count mismatch");
    Matrix out(k_rows.rows, k_cols.rows);
    if (out.rows == 0 || out.cols == 0) return out;
    detail::DevBuf kr = detail::upload({&k_rows}, EMS_F32), vr = detail::upload({&v_rows}, EMS_F32);
    detail::DevBuf kc = detail::upload({&k_cols}, EMS_F32), vc = detail::upload({&v_cols}, EMS_F32);
    detail::DevBuf r(out.rows * out.cols * 4);
    detail::check(ems_redundancy_cross(EMS_F32, static_cast<int32_t>(k_rows.cols), kr.p, vr.p,
                                       static_cast<int32_t>(out.rows), kc.p, vc.p,
                                       static_cast<int32_t>(out.cols), key_only, r.as<float>(), nullptr));
    const auto h = detail::download_raw<float>(r.p, out.rows * out.cols);
    std::copy(h.begin(), h.end(), out.data.begin());
    return out;
}

// sparsity_rate, proj/include/ems/analysis.hpp:22-25 (analysis.cpp:71-91), on the device
// (diag.cu).  The score is rounded to fp32, the device score precision (contract D9).
inline double sparsity_rate(const Vector& score, double zeta) {
    if (score.empty()) throw std::invalid_argument("sparsity_rate: empty score");
    const int32_t n = static_cast<int32_t>(score.size());
    std::vector<float> h(score.begin(), score.end());
    detail::DevBuf s(h.size() * 4), rate(8), ws(ems_diagnostics_workspace_bytes(1, n));
    detail::cuda(cudaMemcpy(s.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    // glo = loc = score: align = 1 and the combined score is the score itself
    detail::check(ems_sparsity_rate(1, n, s.as<float>(), s.as<float>(), zeta, rate.as<double>(), ws.p, ws.n,
                                    nullptr));
    detail::check(ems_sync_status(nullptr, ws.p, nullptr));
    return detail::download_raw<double>(rate.p, 1)[0];
}

// redundancy_rate_direct, proj/include/ems/analysis.hpp (analysis.cpp:93-118), on the device.
inline double redundancy_rate_direct(const Matrix& k_raw, const Matrix& v_raw, double tau, int dtype = EMS_F32) {
    if (k_raw.rows != v_raw.rows || k_raw.rows == 0)
        throw std::invalid_argument("redundancy_rate_direct: bad token count");
    const int32_t n = static_cast<int32_t>(k_raw.rows);
    detail::DevBuf k = detail::upload({&k_raw}, dtype), v = detail::upload({&v_raw}, dtype);
    detail::DevBuf rate(8), ws(ems_diagnostics_workspace_bytes(1, n));
    detail::check(ems_redundancy_rate(dtype, static_cast<int32_t>(k_raw.cols), 1, n, k.p, v.p, tau,
                                      rate.as<double>(), ws.p, ws.n, nullptr));
    return detail::download_raw<double>(rate.p, 1)[0];
}

// engine::prefill's per-head work (proj/src/engine.cpp:65-76) for pre-rotated
// blocks: score + attention on (q_rot, k_rot, v), compress on (k_raw, v).
// With GQA (q_rot.size() = G * k_raw.size()) the KV head's scores are the mean of
// its G query heads' scores (contract D2).
struct PrefillResult {
    std::vector<Matrix> outputs;       // per query head
    std::vector<HeadCacheState> heads; // per KV head
    bool compression_applied = false;
};
inline PrefillResult prefill(const std::vector<Matrix>& q_rot, const std::vector<Matrix>& k_rot,
                             const std::vector<Matrix>& k_raw, const std::vector<Matrix>& v,
                             const CompressionConfig& config, int dtype = EMS_F32) {
    if (k_rot.empty() || k_rot.size() != k_raw.size() || k_raw.size() != v.size() ||
        q_rot.size() % k_rot.size() != 0)
        throw std::invalid_argument("prefill: head count mismatch");
    const std::size_t G = q_rot.size() / k_rot.size(), n = k_rot[0].rows;
    if (n == 0) throw std::invalid_argument("prefill: empty prompt");
    PrefillResult res;
    for (std::size_t h = 0; h < k_rot.size(); ++h) {
        std::vector<const Matrix*> qs;
        for (std::size_t g = 0; g < G; ++g) qs.push_back(&q_rot[h * G + g]);
        std::vector<Matrix> outs;
        Vector glo, loc;
        detail::score_group(qs, k_rot[h], &v[h], std::min(config.l_win, n), dtype, &outs, glo, loc);
        for (auto& o : outs) res.outputs.push_back(std::move(o));
        res.heads.push_back(detail::compress_device(k_raw[h], v[h], glo, loc, config, dtype).cache);
    }
    res.compression_applied = !res.heads.empty() && res.heads[0].compressed;
    return res;
}

}  // namespace ems_b200
