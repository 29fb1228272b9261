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
    std::size_t window_fill = 0;
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
class StateError : public std::runtime_error {  // proj/include/ems/errors.hpp
   public:
    explicit StateError(const std::string& w) : std::runtime_error(w) {}
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
        case EMS_UNSUPPORTED: throw std::invalid_argument(msg);
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
                                      int policy = EMS_POLICY_EMS, std::size_t sink_count = 4,
                                      std::int64_t first_position = 0) {
    const std::size_t n = k_raw.rows, d = k_raw.cols;
    if (n == 0 || v_raw.rows != n || glo.size() != n || loc.size() != n)
        throw std::invalid_argument("compress_prefill: inconsistent token counts");
    ems_desc desc = make_desc(1, 1, n, d, dtype, c);
    desc.first_position = first_position;
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

// compress_prefill, proj/include/ems/compressor.hpp:58-60: token i has logical position
// first_position + i.  dtype (trailing, not in the reference) selects the device precision of K/V.
inline HeadCacheState compress_prefill(const Matrix& k_raw, const Matrix& v_raw,
                                       const ScoreState& scores, const CompressionConfig& config,
                                       std::int64_t first_position = 0, int dtype = EMS_F32) {
    Vector loc(scores.size());
    for (std::size_t i = 0; i < loc.size(); ++i)
        loc[i] = scores.loc_past[i] + (scores.loc_cur.empty() ? 0.0 : scores.loc_cur[i]);
    return detail::compress_device(k_raw, v_raw, scores.glo, loc, config, dtype, EMS_POLICY_EMS, 4, first_position)
        .cache;
}

// effective_score, proj/include/ems/scoring.hpp:66 (scoring.cpp:146-152): mean_pool_1d(
// combine_glo_loc(glo, loc_past + loc_cur), kernel_size) on the device (fp32 scores, D9).
inline Vector effective_score(const ScoreState& state, std::size_t kernel_size) {
    const std::size_t n = state.size();
    if (state.loc_past.size() != n || (!state.loc_cur.empty() && state.loc_cur.size() != n))
        throw std::invalid_argument("combine_glo_loc: length mismatch");
    if (kernel_size % 2 == 0 || kernel_size == 0) throw std::invalid_argument("mean_pool_1d: kernel_size must be odd");
    if (kernel_size > n) throw std::invalid_argument("mean_pool_1d: kernel_size exceeds input length");
    std::vector<float> g(state.glo.begin(), state.glo.end()), lp(state.loc_past.begin(), state.loc_past.end());
    std::vector<float> lc(state.loc_cur.begin(), state.loc_cur.end());
    detail::DevBuf dg(n * 4), dlp(n * 4), dlc(lc.empty() ? 0 : n * 4), out(n * 4), ws(256);
    detail::cuda(cudaMemcpy(dg.p, g.data(), n * 4, cudaMemcpyHostToDevice));
    detail::cuda(cudaMemcpy(dlp.p, lp.data(), n * 4, cudaMemcpyHostToDevice));
    if (!lc.empty()) detail::cuda(cudaMemcpy(dlc.p, lc.data(), n * 4, cudaMemcpyHostToDevice));
    detail::check(ems_effective_score(1, static_cast<int32_t>(n), static_cast<int32_t>(kernel_size), dg.as<float>(),
                                      dlp.as<float>(), lc.empty() ? nullptr : dlc.as<float>(), out.as<float>(), ws.p,
                                      ws.n, nullptr));
    detail::check(ems_sync_status(nullptr, ws.p, nullptr));
    const auto h = detail::download_raw<float>(out.p, n);
    return Vector(h.begin(), h.end());
}

// partition_tokens, proj/include/ems/compressor.hpp:25 (compressor.cpp:48-74), on the device
// select kernels: (score desc, index asc) decided on the fp32 values of pooled_score.
inline TokenPartition partition_tokens(const Vector& pooled_score, const CompressionConfig& config) {
    const std::size_t n = pooled_score.size();
    if (n < config.l_win + 1) throw std::invalid_argument("partition_tokens: need more tokens than the local window");
    ems_desc desc = detail::make_desc(1, 1, n, 1, EMS_F32, config);
    desc.head_dim = 8;  // unused by the partition; any supported head_dim
    detail::check(ems_validate(&desc));
    ems_cache_dims dims{};
    detail::check(ems_cache_dims_for(&desc, &dims));
    const std::size_t C = std::max(dims.centers, 1), T = std::max(dims.tbm, 1);
    std::vector<float> h(pooled_score.begin(), pooled_score.end());
    detail::DevBuf dp(n * 4), pooled(n * 4), cls(n), imp(C * 4), tbm(T * 4), pc(16), dest(T * 4);
    detail::cuda(cudaMemcpy(dp.p, h.data(), n * 4, cudaMemcpyHostToDevice));
    ems_stage stage{pooled.as<float>(), cls.as<int8_t>(), imp.as<int32_t>(), tbm.as<int32_t>(), pc.as<int32_t>(),
                    dest.as<int32_t>()};
    detail::DevBuf ws(ems_workspace_bytes(&desc));
    detail::check(ems_partition(&desc, dp.as<float>(), &stage, ws.p, ws.n, nullptr));
    detail::check(ems_sync_status(&desc, ws.p, nullptr));
    const auto c = detail::download_raw<int8_t>(cls.p, n);
    TokenPartition p;
    for (std::size_t i = 0; i < n; ++i) {
        if (c[i] == 2) p.important.push_back(i);
        else if (c[i] == 1) p.tbm.push_back(i);
        else if (c[i] == 0) p.irrelevant.push_back(i);
        else p.local.push_back(i);
    }
    return p;
}

// assign_merge_destinations, proj/include/ems/compressor.hpp:29 (compressor.cpp:76-95).
inline std::vector<std::int32_t> assign_merge_destinations(const Matrix& r_tbm_to_centers, double tau) {
    const std::size_t R = r_tbm_to_centers.rows, C = r_tbm_to_centers.cols;
    std::vector<std::int32_t> dest(R, kZeroClass);
    if (R == 0 || C == 0) return dest;
    std::vector<float> h(r_tbm_to_centers.data.begin(), r_tbm_to_centers.data.end());
    detail::DevBuf dr(h.size() * 4), dd(R * 4);
    detail::cuda(cudaMemcpy(dr.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    detail::check(ems_assign_merge_destinations(static_cast<int32_t>(R), static_cast<int32_t>(C), dr.as<float>(), tau,
                                                dd.as<int32_t>(), nullptr));
    return detail::download_raw<int32_t>(dd.p, R);
}

// TbmTokens + weighted_merge, proj/include/ems/compressor.hpp:32-51 (compressor.cpp:97-161): the
// merge arithmetic in fp64 on the device (ems_weighted_merge); the LUT entries are appended here in
// the reference's order (zero-class rows first, in row order, only in zero_class mode; then each
// column's members in row order).
struct TbmTokens {
    Matrix k_raw;
    Matrix v_raw;
    std::vector<std::int64_t> positions;
    Vector weights;
    std::vector<ScoreTriple> score_triples;
};
inline void weighted_merge(HeadCacheState& cache, const std::vector<std::int32_t>& center_slot_by_column,
                           const Vector& center_weights, const TbmTokens& tbm,
                           const std::vector<std::int32_t>& destinations, const CompressionConfig& config) {
    if (destinations.size() != tbm.positions.size())
        throw std::invalid_argument("weighted_merge: destination count mismatch");
    const std::size_t n_cols = center_slot_by_column.size(), n_tbm = destinations.size(), d = cache.head_dim;
    if (center_weights.size() != n_cols || tbm.weights.size() != n_tbm || tbm.score_triples.size() != n_tbm ||
        tbm.k_raw.rows != n_tbm || tbm.v_raw.rows != n_tbm || (n_tbm && (tbm.k_raw.cols != d || tbm.v_raw.cols != d)))
        throw std::invalid_argument("weighted_merge: inconsistent sizes");
    std::vector<std::vector<std::size_t>> members(n_cols);
    for (std::size_t i = 0; i < n_tbm; ++i) {
        const std::int32_t c = destinations[i];
        if (c == kZeroClass) {
            if (config.eviction == EvictionRealization::zero_class) cache.lut.push_back({tbm.positions[i], kZeroClass});
            continue;
        }
        if (c < 0 || static_cast<std::size_t>(c) >= n_cols) throw std::invalid_argument("weighted_merge: bad destination");
        members[static_cast<std::size_t>(c)].push_back(i);
    }
    std::vector<double> uk(n_cols * d), val(n_cols * d), sc(n_cols * 3), tk(n_tbm * d), tv(n_tbm * d), ts(n_tbm * 3);
    for (std::size_t c = 0; c < n_cols; ++c) {
        const std::int32_t slot = center_slot_by_column[c];
        if (slot < 0 || static_cast<std::size_t>(slot) >= cache.slots.size() || !cache.slots[slot])
            throw CorruptionError("weighted_merge: column names a nonexistent slot");
        const CenterEntry& e = *cache.slots[slot];
        std::copy(e.unit_key.begin(), e.unit_key.end(), uk.begin() + c * d);
        std::copy(e.value.begin(), e.value.end(), val.begin() + c * d);
        sc[3 * c] = e.score.glo, sc[3 * c + 1] = e.score.loc_past, sc[3 * c + 2] = e.score.loc_cur;
    }
    for (std::size_t i = 0; i < n_tbm; ++i) {
        std::copy(tbm.k_raw.data.begin() + i * d, tbm.k_raw.data.begin() + (i + 1) * d, tk.begin() + i * d);
        std::copy(tbm.v_raw.data.begin() + i * d, tbm.v_raw.data.begin() + (i + 1) * d, tv.begin() + i * d);
        const ScoreTriple& t = tbm.score_triples[i];
        ts[3 * i] = t.glo, ts[3 * i + 1] = t.loc_past, ts[3 * i + 2] = t.loc_cur;
    }
    auto up = [](const std::vector<double>& h) {
        detail::DevBuf b(h.size() * 8);
        if (!h.empty()) detail::cuda(cudaMemcpy(b.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
        return b;
    };
    detail::DevBuf duk = up(uk), dval = up(val), dsc = up(sc), dcw = up(center_weights), dtk = up(tk), dtv = up(tv),
                   dtw = up(tbm.weights), dts = up(ts), ddest(n_tbm * 4);
    if (n_tbm) detail::cuda(cudaMemcpy(ddest.p, destinations.data(), n_tbm * 4, cudaMemcpyHostToDevice));
    detail::check(ems_weighted_merge(static_cast<int32_t>(d), static_cast<int32_t>(n_cols), duk.as<double>(),
                                     dval.as<double>(), dsc.as<double>(), dcw.as<double>(), static_cast<int32_t>(n_tbm),
                                     dtk.as<double>(), dtv.as<double>(), dtw.as<double>(), dts.as<double>(),
                                     ddest.as<int32_t>(), nullptr));
    const auto uk2 = detail::download_raw<double>(duk.p, uk.size()), val2 = detail::download_raw<double>(dval.p, val.size());
    const auto sc2 = detail::download_raw<double>(dsc.p, sc.size());
    for (std::size_t c = 0; c < n_cols; ++c) {
        if (members[c].empty()) continue;  // untouched, bit for bit
        const std::int32_t slot = center_slot_by_column[c];
        CenterEntry& e = *cache.slots[slot];
        e.unit_key.assign(uk2.begin() + c * d, uk2.begin() + (c + 1) * d);
        e.value.assign(val2.begin() + c * d, val2.begin() + (c + 1) * d);
        e.score = {sc2[3 * c], sc2[3 * c + 1], sc2[3 * c + 2]};
        for (std::size_t i : members[c]) cache.lut.push_back({tbm.positions[i], slot});
    }
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

// engine::prefill's per-head work (proj/src/engine.cpp:65-76) for PRE-ROTATED blocks with GQA:
// score + attention on (q_rot, k_rot, v), compress on (k_raw, v).  With q_rot.size() = G *
// k_raw.size() the KV head's scores are the mean of its G query heads' scores (contract D2).
// (The reference's own engine entry point, on raw blocks with RoPE inside, is prefill(EngineState&,
// ...) below.)
struct RotatedPrefillResult {
    std::vector<Matrix> outputs;        // per query head
    std::vector<HeadCacheState> heads;  // per KV head
    bool compression_applied = false;
};
inline RotatedPrefillResult prefill_rotated(const std::vector<Matrix>& q_rot, const std::vector<Matrix>& k_rot,
                                            const std::vector<Matrix>& k_raw, const std::vector<Matrix>& v,
                                            const CompressionConfig& config, int dtype = EMS_F32) {
    if (k_rot.empty() || k_rot.size() != k_raw.size() || k_raw.size() != v.size() ||
        q_rot.size() % k_rot.size() != 0)
        throw std::invalid_argument("prefill: head count mismatch");
    const std::size_t G = q_rot.size() / k_rot.size(), n = k_rot[0].rows;
    if (n == 0) throw std::invalid_argument("prefill: empty prompt");
    RotatedPrefillResult res;
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

// ---------------------------------------------------------------- engine.hpp (prefill)
struct RopeParams {  // proj/include/ems/rope.hpp:9-12
    std::size_t head_dim = 0;
    double base = 10000.0;
};
struct AttentionOutput {  // proj/include/ems/engine.hpp:14-18
    Matrix outputs;
    bool weights_available = false;
    Matrix weights;
};
struct EngineState {  // proj/include/ems/engine.hpp:22-31
    std::size_t num_heads = 0;
    std::size_t head_dim = 0;
    CompressionConfig config;
    PolicyHandle policy;
    RopeParams rope;
    std::vector<HeadCacheState> heads;
    std::int64_t next_position = 0;
    bool prefilled = false;
    int dtype = EMS_F32;  // device precision of Q/K/V (not in the reference)
};
struct PrefillResult {  // proj/include/ems/engine.hpp:36-39
    std::vector<AttentionOutput> per_head;
    bool compression_applied = false;
};

// make_engine, proj/src/engine.cpp:26-40.
inline EngineState make_engine(std::size_t num_heads, std::size_t head_dim, PolicyHandle policy,
                               CompressionConfig config, double rope_base = 10000.0) {
    if (num_heads == 0 || head_dim == 0 || head_dim % 2 != 0)
        throw std::invalid_argument("make_engine: need heads >= 1 and even head_dim");
    policy.validate(config);
    EngineState s;
    s.num_heads = num_heads;
    s.head_dim = head_dim;
    s.config = config;
    s.policy = policy;
    s.rope = RopeParams{head_dim, rope_base};
    s.heads.resize(num_heads);
    return s;
}

// prefill, proj/include/ems/engine.hpp:44-45 (engine.cpp:42-82): RAW per-head blocks; RoPE
// (positions 0..n-1), causal attention with the Global-Local score, init_score_state and the
// policy's prefill compression run on the device for all heads in one ems_prefill call.
inline PrefillResult prefill(EngineState& state, const std::vector<Matrix>& q_blocks,
                             const std::vector<Matrix>& k_blocks, const std::vector<Matrix>& v_blocks) {
    if (q_blocks.size() != state.num_heads || k_blocks.size() != state.num_heads ||
        v_blocks.size() != state.num_heads)
        throw std::invalid_argument("prefill: head count mismatch");
    const std::size_t n = q_blocks[0].rows, d = state.head_dim, H = state.num_heads;
    if (n == 0) throw std::invalid_argument("prefill: empty prompt");
    for (std::size_t h = 0; h < H; ++h)
        if (q_blocks[h].rows != n || k_blocks[h].rows != n || v_blocks[h].rows != n)
            throw std::invalid_argument("prefill: token count mismatch across blocks");
    if (state.prefilled) throw StateError("prefill: engine already prefilled");
    for (std::size_t h = 0; h < H; ++h)
        if (q_blocks[h].cols != d || k_blocks[h].cols != d || v_blocks[h].cols != d)
            throw std::invalid_argument("prefill: head_dim mismatch");
    const int dtype = state.dtype;
    ems_desc desc = detail::make_desc(H, H, n, d, dtype, state.config);
    desc.policy = policy_code(state.policy.kind);
    desc.sink_count = static_cast<int32_t>(state.policy.sink_count);
    detail::check(ems_validate(&desc));
    ems_cache_dims dims{};
    detail::check(ems_cache_dims_for(&desc, &dims));
    std::vector<const Matrix*> qs, ks, vs;
    for (std::size_t h = 0; h < H; ++h) qs.push_back(&q_blocks[h]), ks.push_back(&k_blocks[h]), vs.push_back(&v_blocks[h]);
    detail::DevBuf dq = detail::upload(qs, dtype), dk = detail::upload(ks, dtype), dv = detail::upload(vs, dtype);
    const std::size_t es = dtype == EMS_F32 ? 4 : 2;
    detail::DevBuf dqr(H * n * d * es), dkr(H * n * d * es), dout(H * n * d * es);
    const std::size_t C = dims.centers, Lc = dims.locals, U = std::max(dims.lut, 1);
    detail::DevBuf ck(H * C * d * es), cn(H * C * 4), cv(H * C * d * es), cp(H * C * 4), cs(H * C * 12),
        lk(H * Lc * d * es), lv(H * Lc * d * es), lp(H * Lc * 4), ls(H * Lc * 12), up(H * U * 4), us(H * U * 4),
        cnt(H * 16);
    ems_cache cache{ck.p, cn.as<float>(), cv.p, cp.as<int32_t>(), cs.as<float>(), lk.p, lv.p,
                    lp.as<int32_t>(), ls.as<float>(), up.as<int32_t>(), us.as<int32_t>(), cnt.as<int32_t>()};
    detail::DevBuf ws(ems_workspace_bytes(&desc));
    detail::check(ems_prefill(&desc, state.rope.base, dq.p, dk.p, dv.p, dqr.p, dkr.p, dout.p, nullptr, nullptr,
                              nullptr, nullptr, &cache, ws.p, ws.n, nullptr));
    detail::check(ems_sync_status(&desc, ws.p, nullptr));
    PrefillResult result;
    const auto o = detail::download(dout.p, H * n * d, dtype);
    result.per_head.resize(H);
    const auto counts = detail::download_raw<int32_t>(cnt.p, H * 4);
    const auto ckh = detail::download(ck.p, H * C * d, dtype), cvh = detail::download(cv.p, H * C * d, dtype);
    const auto cnh = detail::download_raw<float>(cn.p, H * C), csh = detail::download_raw<float>(cs.p, H * C * 3);
    const auto cph = detail::download_raw<int32_t>(cp.p, H * C);
    const auto lkh = detail::download(lk.p, H * Lc * d, dtype), lvh = detail::download(lv.p, H * Lc * d, dtype);
    const auto lph = detail::download_raw<int32_t>(lp.p, H * Lc);
    const auto lsh = detail::download_raw<float>(ls.p, H * Lc * 3);
    const auto uph = detail::download_raw<int32_t>(up.p, H * U), ush = detail::download_raw<int32_t>(us.p, H * U);
    for (std::size_t h = 0; h < H; ++h) {
        result.per_head[h].outputs = Matrix(n, d);
        std::copy(o.begin() + h * n * d, o.begin() + (h + 1) * n * d, result.per_head[h].outputs.data.begin());
        HeadCacheState hc;
        hc.head_dim = d;
        hc.compressed = counts[4 * h + 3] != 0;
        for (int s = 0; s < counts[4 * h]; ++s) {
            const std::size_t e = h * C + s;
            CenterEntry c;
            c.unit_key.assign(ckh.begin() + e * d, ckh.begin() + (e + 1) * d);
            c.value.assign(cvh.begin() + e * d, cvh.begin() + (e + 1) * d);
            c.key_norm = cnh[e];
            c.position = cph[e];
            c.score = {csh[3 * e], csh[3 * e + 1], csh[3 * e + 2]};
            hc.slots.emplace_back(std::move(c));
        }
        for (int i = 0; i < counts[4 * h + 1]; ++i) {
            const std::size_t e = h * Lc + i;
            LocalEntry l;
            l.key.assign(lkh.begin() + e * d, lkh.begin() + (e + 1) * d);
            l.value.assign(lvh.begin() + e * d, lvh.begin() + (e + 1) * d);
            l.position = lph[e];
            l.score = {lsh[3 * e], lsh[3 * e + 1], lsh[3 * e + 2]};
            hc.locals.push_back(std::move(l));
        }
        for (int i = 0; i < counts[4 * h + 2]; ++i) hc.lut.push_back({uph[h * U + i], ush[h * U + i]});
        hc.window_fill = 0;
        state.heads[h] = std::move(hc);
    }
    state.next_position = static_cast<std::int64_t>(n);
    state.prefilled = true;
    result.compression_applied = state.heads[0].compressed;
    return result;
}

}  // namespace ems_b200
