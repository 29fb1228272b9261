// capi.cu -- the extern "C" boundary (include/ems_b200.h): validation, workspace
// layout and the launch sequence of the four kernels.  No allocation, no host
// synchronisation on the hot path; everything is stream-ordered.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ems {

cudaError_t score_simt(const Dims& dm, int dtype, const void* q, const void* k, const void* v,
                       void* o, float* lse, float* glo, float* loc, cudaStream_t s);
cudaError_t score_tc(const Dims& dm, const void* q, const void* k, const void* v, void* o,
                     float* lse, float* glo, float* loc, void* ws, cudaStream_t s, cudaEvent_t o_ready,
                     const ScoreParts* parts);
size_t score_tc_workspace(const Dims& dm);
size_t merge_tc_workspace(const Dims& dm);
bool merge_tc_supported(const Dims& dm, int dtype);
cudaError_t launch_merge_tc(const Dims& dm, const void* k, const void* v, const ems_stage& sg,
                            double tau, int key_only, void* ws, cudaStream_t s);
bool score_tc_supported(const Dims& dm, int dtype);
cudaError_t launch_select(const Dims& dm, int l_win, int n_imp, int n_tbm, int kernel,
                          const float* glo, const float* loc, const ems_stage& sg,
                          DevStatus* status, cudaStream_t s, int policy, int sink, int n_budget);
cudaError_t launch_merge_assign(const Dims& dm, int dtype, const void* k, const void* v,
                                const ems_stage& sg, double tau, int key_only, float* inv_kc,
                                float* inv_vc, float* inv_kt, float* inv_vt, cudaStream_t s);
cudaError_t launch_merge_scatter(const Dims& dm, int dtype, const void* k, const void* v,
                                 const float* glo, const float* loc, const ems_stage& sg,
                                 int32_t* ws_count, int32_t* ws_members, const ems_cache& cache,
                                 DevStatus* status, cudaStream_t s);
cudaError_t launch_compact(const Dims& dm, int dtype, const void* k, const void* v,
                           const float* glo, const float* loc, const ems_stage& sg,
                           const ems_cache& c, int zero_class, int64_t first_pos, DevStatus* status,
                           cudaStream_t s);
cudaError_t launch_keep_all(const Dims& dm, int dtype, const void* k, const void* v,
                            const float* glo, const float* loc, const ems_stage& sg,
                            const ems_cache& c, int64_t first_pos, cudaStream_t s);
cudaError_t launch_rope(int dtype, int planes, int L, int d, double base, long long first_pos,
                        const void* x, void* y, cudaStream_t s);
cudaError_t launch_rope_table(float2* table, int max_pos, int d, double base, cudaStream_t s);
size_t rope_table64_bytes(int L, int d);
cudaError_t launch_rope_table64(void* tab, int L, int d, double base, long long first_pos, cudaStream_t s);
cudaError_t launch_rope_tab(int dtype, int planes, int L, int d, const void* tab, const void* x, void* y,
                            cudaStream_t s);
cudaError_t launch_decode_init(const Dims& m, int dtype, const ems_cache& c, const ems_decode_state& st,
                               int S, int W, int T, cudaStream_t s);
cudaError_t launch_decode_step(const Dims& m, int dtype, int S, int W, int T, int R, int l_win, int lut_cap,
                               double tau, int zero_class, int with_pos, long long position, int max_pos,
                               const float2* table, const void* q, const void* k, const void* v, void* out,
                               int32_t* argmax_pos, const ems_decode_state& st, void* ws, cudaStream_t s,
                               int policy, int sink, int n_budget);
size_t decode_workspace_bytes(const Dims& m, int R);
size_t decode_smem_bytes(const Dims& m, int S, int W);
cudaError_t launch_redundancy_cross(int dtype, int d, const void* kr, const void* vr, int nr,
                                    const void* kc, const void* vc, int nc, int key_only,
                                    float* r, cudaStream_t s);
size_t diag_workspace_bytes(int units, int L);
cudaError_t launch_effective_score(int units, int L, int kernel, const float* glo, const float* loc_past,
                                   const float* loc_cur, float* pooled, DevStatus* status, cudaStream_t s);
cudaError_t launch_assign_rows(const float* r, int n_rows, int n_cols, double tau, int32_t* dest, cudaStream_t s);
cudaError_t launch_weighted_merge(int d, int n_cols, double* uk, double* val, double* score, const double* cw,
                                  int n_tbm, const double* tk, const double* tv, const double* tw, const double* ts,
                                  const int32_t* dest, cudaStream_t s);
cudaError_t launch_sparsity(int units, int L, const float* glo, const float* loc, double zeta, double* rate,
                            void* ws, int unit_base, cudaStream_t s);
cudaError_t launch_redundancy(int units, int L, int d, int dtype, const void* k, const void* v, double tau,
                              double* rate, void* ws, cudaStream_t s);

namespace {
thread_local char g_err[1024] = "";
}

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

cudaError_t smem_optin(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes opted in
    if (bytes <= 48 * 1024) return cudaSuccess;              // always available without opt-in
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int& have = done[{kernel, dev}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

int active_clusters(const void* kernel, int threads, int smem_bytes, int cluster) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> clusters
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(mu);
    int& have = done[{kernel, dev}];
    if (have > 0) return have;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cluster, 1, 1);
    cfg.blockDim = dim3((unsigned)threads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem_bytes;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        n = sms / cluster;  // one CTA per SM
    }
    have = n;
    return n;
}

Dims make_dims(const ems_desc& d) {
    Dims m;
    m.B = d.batch;
    m.Hq = d.heads_q;
    m.Hkv = d.heads_kv;
    m.G = d.heads_kv > 0 ? d.heads_q / d.heads_kv : 0;
    m.L = d.seq_len;
    m.d = d.head_dim;
    m.units = d.batch * d.heads_kv;
    m.lwin_scores = d.l_win < d.seq_len ? d.l_win : d.seq_len;  // engine.cpp:63
    m.cap_c = d.n_budget - d.l_win;                                // cache.hpp:32
    m.cap_l = d.policy == EMS_POLICY_FULL && d.seq_len > d.n_budget ? d.seq_len : d.n_budget;
    // cache.hpp:33-35; the baseline policies never merge (policies.cpp:49-75)
    m.cap_tbm = d.policy == EMS_POLICY_EMS ? (int)((d.gamma - 1.0) * (double)d.n_budget) : 0;
    m.cap_lut = m.cap_c + m.cap_tbm;
    m.esize = d.dtype == EMS_F32 ? 4 : 2;
    return m;
}

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Workspace carve-up.  Offsets are deterministic functions of the descriptor.
struct Layout {
    size_t status, lse, glo, loc, pooled, cls, imp, tbm, pcount, dest, inv, cnt, mem, tc, mtc, total;
};

Layout layout(const ems_desc& d) {
    const Dims m = make_dims(d);
    Layout l{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += align_up(bytes);
        return o;
    };
    const size_t U = (size_t)m.units, L = (size_t)m.L;
    l.status = take(sizeof(DevStatus));
    l.lse = take(sizeof(float) * (size_t)m.B * m.Hq * L);
    l.glo = take(sizeof(float) * U * L);
    l.loc = take(sizeof(float) * U * L);
    l.pooled = take(sizeof(float) * U * L);
    l.cls = take(U * L);
    l.imp = take(sizeof(int32_t) * U * (size_t)m.cap_c);
    l.tbm = take(sizeof(int32_t) * U * (size_t)(m.cap_tbm > 0 ? m.cap_tbm : 1));
    l.pcount = take(sizeof(int32_t) * U * 4);
    l.dest = take(sizeof(int32_t) * U * (size_t)(m.cap_tbm > 0 ? m.cap_tbm : 1));
    l.inv = take(sizeof(float) * U * 2 * (size_t)(m.cap_c + m.cap_tbm));
    l.cnt = take(sizeof(int32_t) * U * (size_t)(m.cap_c + 1));
    l.mem = take(sizeof(int32_t) * U * (size_t)(m.cap_tbm > 0 ? m.cap_tbm : 1));
    l.tc = take(score_tc_workspace(m));
    l.mtc = take(merge_tc_supported(m, d.dtype) ? merge_tc_workspace(m) : 0);
    l.total = off;
    return l;
}

template <class P>
P* at(void* ws, size_t off) {
    return reinterpret_cast<P*>(static_cast<char*>(ws) + off);
}

ems_stage default_stage(const ems_desc& d, void* ws) {
    const Layout l = layout(d);
    ems_stage s;
    s.pooled = at<float>(ws, l.pooled);
    s.cls = at<int8_t>(ws, l.cls);
    s.imp_idx = at<int32_t>(ws, l.imp);
    s.tbm_idx = at<int32_t>(ws, l.tbm);
    s.part_counts = at<int32_t>(ws, l.pcount);
    s.dest = at<int32_t>(ws, l.dest);
    return s;
}

// The whole problem, and any contiguous group of its units as the chunked host pipeline runs
// them (ems_prefill_host): a group's score workspace can exceed its share of the whole one
// (colsum head-split partials), so the requirement is the maximum over group sizes.
size_t workspace_need(const ems_desc& d) {
    size_t need = layout(d).total;
    const int G = d.heads_q / d.heads_kv, U = d.batch * d.heads_kv;
    for (int n = 1; n < U; ++n) {
        ems_desc sub = d;
        sub.batch = 1;
        sub.heads_kv = n;
        sub.heads_q = n * G;
        const size_t t = layout(sub).total;
        if (t > need) need = t;
    }
    return need;
}

int check_ws(const ems_desc* d, void* ws, size_t bytes) {
    const size_t need = workspace_need(*d);
    if (ws == nullptr || bytes < need) {
        set_error("workspace too small: need %zu bytes, got %zu", need, bytes);
        return EMS_INVALID_ARGUMENT;
    }
    if (reinterpret_cast<uintptr_t>(ws) % 16 != 0) {
        set_error("workspace must be 16-byte aligned");
        return EMS_INVALID_ARGUMENT;
    }
    return EMS_OK;
}

bool supported_dim(int d) {
    return d == 8 || d == 16 || d == 32 || d == 64 || d == 96 || d == 128;
}

int kernel_eff(const ems_desc& d) {  // clamp_kernel, compressor.cpp:29-34
    if (d.kernel_size <= d.seq_len) return d.kernel_size;
    return (d.seq_len % 2 == 1) ? d.seq_len : d.seq_len - 1;
}

bool use_tc(const ems_desc& d) {
    const Dims m = make_dims(d);
    if (d.score_impl == EMS_SCORE_SIMT) return false;
    return score_tc_supported(m, d.dtype);
}

// o_ready (optional) is recorded on `s` as soon as O and the LSE are final: after the forward
// pass, before the column sums of the tensor-core path.
int run_score(const ems_desc* desc, const void* q, const void* k, const void* v, void* o,
              float* lse, float* glo, float* loc, void* ws, cudaStream_t s, cudaEvent_t o_ready = nullptr,
              const ScoreParts* parts = nullptr) {
    const Dims m = make_dims(*desc);
    const Layout l = layout(*desc);
    float* lse_buf = lse ? lse : at<float>(ws, l.lse);
    cudaError_t e;
    if (use_tc(*desc)) {
        e = score_tc(m, q, k, v, o, lse_buf, glo, loc, at<void>(ws, l.tc), s, o_ready, parts);
    } else {
        // The SIMT kernels serve fp32 (no tcgen05 kind keeps the 1e-4 contract) and head_dim
        // != 128; bf16 at d = 128 always takes the tensor cores (any L up to 2^20) unless the
        // caller asks for the SIMT twin explicitly -- never a silent ~700x slower path.
        const bool tc_shape = desc->dtype == EMS_BF16 && desc->head_dim == 128;
        if (desc->score_impl == EMS_SCORE_TCGEN05 || (tc_shape && desc->score_impl == EMS_SCORE_AUTO)) {
            set_error("tcgen05 score pass unavailable (needs an sm_100 device and seq_len <= 1048576; "
                      "got seq_len %d)", desc->seq_len);
            return EMS_UNSUPPORTED;
        }
        e = cudaSuccess;
        if (parts)
            for (int p = 0; p < parts->n && e == cudaSuccess; ++p) e = parts->before(p, s);
        if (e == cudaSuccess) e = score_simt(m, desc->dtype, q, k, v, o, lse_buf, glo, loc, s);
        if (e == cudaSuccess && o_ready) e = cudaEventRecord(o_ready, s);
    }
    if (e != cudaSuccess) {
        set_error("score launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int run_select(const ems_desc* desc, const float* glo, const float* loc, const ems_stage& sg,
               void* ws, cudaStream_t s, int unit_base = 0, bool pooled_given = false) {
    Dims m = make_dims(*desc);
    m.unit_base = unit_base;
    const int n_cand = m.L - desc->l_win;
    int n_imp = m.cap_c < n_cand ? m.cap_c : n_cand;                     // :64
    const int n_tbm = m.cap_tbm < n_cand - n_imp ? m.cap_tbm : n_cand - n_imp;  // :65
    if (desc->policy == EMS_POLICY_STREAMING) {  // policies.cpp:145-159: sinks + recent window
        const long long sink = desc->sink_count < m.L ? desc->sink_count : m.L;
        const long long recent = desc->n_budget - desc->sink_count;
        long long lo = m.L - recent;
        if (lo < desc->sink_count) lo = desc->sink_count;
        n_imp = (int)(sink + (n_cand > lo ? n_cand - lo : 0));
    }
    cudaError_t e = launch_select(m, desc->l_win, n_imp, n_tbm, kernel_eff(*desc), glo, loc, sg,
                                  at<DevStatus>(ws, layout(*desc).status), s,
                                  pooled_given ? kPolicyPooled : desc->policy, desc->sink_count, desc->n_budget);
    if (e != cudaSuccess) {
        set_error("select launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int run_merge(const ems_desc* desc, const void* k_raw, const void* v, const ems_stage& sg,
              void* ws, cudaStream_t s) {
    const Dims m = make_dims(*desc);
    if (m.cap_tbm <= 0) return EMS_OK;
    const Layout l = layout(*desc);
    cudaError_t e;
    // tensor-core similarity for bf16 / d = 128 unless the SIMT kernels are forced
    if (desc->score_impl != EMS_SCORE_SIMT && merge_tc_supported(m, desc->dtype)) {
        e = launch_merge_tc(m, k_raw, v, sg, desc->tau, desc->key_only, at<void>(ws, l.mtc), s);
    } else {
        float* inv = at<float>(ws, l.inv);
        const size_t U = m.units;
        float* inv_kc = inv;
        float* inv_vc = inv_kc + U * m.cap_c;
        float* inv_kt = inv_vc + U * m.cap_c;
        float* inv_vt = inv_kt + U * m.cap_tbm;
        e = launch_merge_assign(m, desc->dtype, k_raw, v, sg, desc->tau, desc->key_only, inv_kc,
                                inv_vc, inv_kt, inv_vt, s);
    }
    if (e != cudaSuccess) {
        set_error("merge launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int run_compact(const ems_desc* desc, const void* k_raw, const void* v, const float* glo,
                const float* loc, const ems_stage& sg, const ems_cache& c, void* ws,
                cudaStream_t s, int unit_base = 0) {
    Dims m = make_dims(*desc);
    m.unit_base = unit_base;
    const Layout l = layout(*desc);
    cudaError_t e;
    if (m.L <= desc->n_budget || desc->policy == EMS_POLICY_FULL) {  // policies.cpp:136-138
        e = launch_keep_all(m, desc->dtype, k_raw, v, glo, loc, sg, c, desc->first_position, s);
    } else {
        ems_stage sg2 = sg;
        if (m.cap_tbm <= 0) sg2.dest = at<int32_t>(ws, l.dest);  // never read (no TBM tokens)
        e = launch_compact(m, desc->dtype, k_raw, v, glo, loc, sg2, c, desc->zero_class,
                           desc->first_position, at<DevStatus>(ws, l.status), s);
        if (e == cudaSuccess && m.cap_tbm > 0) {
            e = launch_merge_scatter(m, desc->dtype, k_raw, v, glo, loc, sg, at<int32_t>(ws, l.cnt),
                                     at<int32_t>(ws, l.mem), c, at<DevStatus>(ws, l.status), s);
            if (e != cudaSuccess) {
                set_error("weighted-merge launch: %s", cudaGetErrorString(e));
                return EMS_CUDA_ERROR;
            }
        }
    }
    if (e != cudaSuccess) {
        set_error("compact launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

}  // namespace
}  // namespace ems

using namespace ems;

extern "C" {

int ems_abi_version(void) { return EMS_B200_ABI_VERSION; }
const char* ems_last_error(void) { return g_err; }

const char* ems_status_string(int status) {
    switch (status) {
        case EMS_OK: return "ok";
        case EMS_INVALID_ARGUMENT: return "invalid argument";
        case EMS_DEGENERATE_INPUT: return "degenerate input";
        case EMS_CORRUPTION: return "corruption";
        case EMS_CUDA_ERROR: return "cuda error";
        case EMS_UNSUPPORTED: return "unsupported";
        default: return "unknown";
    }
}

int ems_validate(const ems_desc* d) {
    if (d == nullptr) {
        set_error("null descriptor");
        return EMS_INVALID_ARGUMENT;
    }
    if (d->batch <= 0 || d->heads_q <= 0 || d->heads_kv <= 0 || d->heads_q % d->heads_kv != 0) {
        set_error("bad head/batch shape (B=%d Hq=%d Hkv=%d)", d->batch, d->heads_q, d->heads_kv);
        return EMS_INVALID_ARGUMENT;
    }
    if (d->seq_len <= 0) {  // prefill: empty prompt (engine.cpp:49-51)
        set_error("empty prompt");
        return EMS_INVALID_ARGUMENT;
    }
    if (!supported_dim(d->head_dim)) {
        set_error("head_dim %d unsupported (8,16,32,64,96,128)", d->head_dim);
        return EMS_INVALID_ARGUMENT;
    }
    if (d->dtype != EMS_F32 && d->dtype != EMS_BF16) {
        set_error("dtype must be EMS_F32 or EMS_BF16");
        return EMS_INVALID_ARGUMENT;
    }
    // CompressionConfig::validate, proj/src/cache.cpp:12-28
    if (d->n_budget <= 0 || d->l_win <= 0 || d->n_budget <= d->l_win) {
        set_error("CompressionConfig: require n_budget > l_win > 0");
        return EMS_INVALID_ARGUMENT;
    }
    if (!(d->tau >= 0.0 && d->tau <= 1.0)) {
        set_error("CompressionConfig: tau must be in [0, 1]");
        return EMS_INVALID_ARGUMENT;
    }
    if (!(d->gamma >= 1.0)) {
        set_error("CompressionConfig: gamma must be >= 1");
        return EMS_INVALID_ARGUMENT;
    }
    if (d->kernel_size <= 0 || d->kernel_size % 2 == 0) {
        set_error("CompressionConfig: kernel_size must be odd");
        return EMS_INVALID_ARGUMENT;
    }
    if (d->score_impl < 0 || d->score_impl > 2) {
        set_error("bad score_impl");
        return EMS_INVALID_ARGUMENT;
    }
    if (d->policy < EMS_POLICY_EMS || d->policy > EMS_POLICY_SNAPKV) {
        set_error("bad policy %d", d->policy);
        return EMS_INVALID_ARGUMENT;
    }
    if (d->policy == EMS_POLICY_STREAMING && (d->sink_count < 0 || d->n_budget < d->sink_count + d->l_win)) {
        set_error("streaming_llm: n_budget must cover sinks plus the local window");  // policies.cpp:113-115
        return EMS_INVALID_ARGUMENT;
    }
    if ((long long)d->seq_len + d->first_position > 0x7fffffffLL || d->first_position < 0) {
        set_error("positions must fit int32");
        return EMS_INVALID_ARGUMENT;
    }
    return EMS_OK;
}

int ems_cache_dims_for(const ems_desc* d, ems_cache_dims* out) {
    if (int rc = ems_validate(d)) return rc;
    const Dims m = make_dims(*d);
    out->units = m.units;
    out->centers = m.cap_c;
    out->locals = m.cap_l;
    out->lut = m.cap_lut;
    out->tbm = m.cap_tbm;
    return EMS_OK;
}

size_t ems_workspace_bytes(const ems_desc* d) {
    if (ems_validate(d) != EMS_OK) return 0;
    return workspace_need(*d);
}

size_t ems_prefill_host_workspace_bytes(const ems_desc* d) {
    if (ems_validate(d) != EMS_OK) return 0;
    // two unit groups in flight + the RoPE (cos, sin) table of the problem
    return 2 * ems::align_up(ems::workspace_need(*d)) + ems::align_up(ems::rope_table64_bytes(d->seq_len, d->head_dim));
}

int ems_score(const ems_desc* d, const void* q, const void* k, const void* v, void* out_o,
              float* lse, float* glo, float* loc, void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_score");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    if (!q || !k || !glo || !loc || (out_o && !v)) {
        set_error("ems_score: null tensor");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));  // start of a pipeline
    return run_score(d, q, k, v, out_o, lse, glo, loc, ws, s);
}

int ems_select(const ems_desc* d, const float* glo, const float* loc, const ems_stage* st,
               void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_select");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    if (d->seq_len <= d->n_budget || d->policy == EMS_POLICY_FULL) {
        set_error("ems_select: keep-all (prompt fits the budget, or the full policy) has no partition");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));
    const ems_stage sg = st ? *st : default_stage(*d, ws);
    return run_select(d, glo, loc, sg, ws, s);
}

int ems_partition(const ems_desc* d, const float* pooled, const ems_stage* st, void* ws, size_t ws_bytes,
                  cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_partition");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    if (!pooled || !st) {
        set_error("ems_partition: null pooled scores or stage");
        return EMS_INVALID_ARGUMENT;
    }
    if (d->seq_len < d->l_win + 1 || d->policy != EMS_POLICY_EMS) {  // compressor.cpp:50-52
        set_error("partition_tokens: need more tokens than the local window (EMS policy)");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));
    return run_select(d, pooled, pooled, *st, ws, s, 0, true);
}

int ems_effective_score(int32_t units, int32_t L, int32_t kernel, const float* glo, const float* loc_past,
                        const float* loc_cur, float* pooled, void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_effective_score");
    if (units < 0 || L < 1 || kernel < 1 || kernel % 2 == 0 || kernel > L) {  // numerics.cpp:63-68
        set_error("effective_score: kernel_size must be odd and <= the input length");
        return EMS_INVALID_ARGUMENT;
    }
    if ((units > 0 && (!glo || !loc_past || !pooled)) || !ws || ws_bytes < sizeof(DevStatus)) {
        set_error("effective_score: null buffer or workspace < %zu bytes", sizeof(DevStatus));
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));
    if (units == 0) return EMS_OK;
    EMS_CUDA_CHECK(launch_effective_score(units, L, kernel, glo, loc_past, loc_cur, pooled,
                                          static_cast<DevStatus*>(ws), s));
    return EMS_OK;
}

int ems_assign_merge_destinations(int32_t n_rows, int32_t n_cols, const float* r, double tau, int32_t* dest,
                                  cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_assign_merge_destinations");
    if (n_rows < 0 || n_cols < 0 || (n_rows > 0 && (!dest || (n_cols > 0 && !r)))) {
        set_error("assign_merge_destinations: bad arguments");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(launch_assign_rows(r, n_rows, n_cols, tau, dest, s));
    return EMS_OK;
}

int ems_weighted_merge(int32_t d, int32_t n_cols, double* center_unit_key, double* center_value,
                       double* center_score, const double* center_weight, int32_t n_tbm, const double* tbm_key,
                       const double* tbm_value, const double* tbm_weight, const double* tbm_score,
                       const int32_t* dest, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_weighted_merge");
    if (d < 1 || d > 512 || n_cols < 0 || n_tbm < 0 ||
        (n_cols > 0 && (!center_unit_key || !center_value || !center_score || !center_weight)) ||
        (n_tbm > 0 && (!tbm_key || !tbm_value || !tbm_weight || !tbm_score || !dest))) {
        set_error("weighted_merge: bad arguments (head_dim in [1, 512], non-null buffers)");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(launch_weighted_merge(d, n_cols, center_unit_key, center_value, center_score, center_weight,
                                         n_tbm, tbm_key, tbm_value, tbm_weight, tbm_score, dest, s));
    return EMS_OK;
}

int ems_merge(const ems_desc* d, const void* k_raw, const void* v, const ems_stage* st, void* ws,
              size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_merge");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    const ems_stage sg = st ? *st : default_stage(*d, ws);
    return run_merge(d, k_raw, v, sg, ws, s);
}

int ems_compact(const ems_desc* d, const void* k_raw, const void* v, const float* glo,
                const float* loc, const ems_stage* st, const ems_cache* c, void* ws,
                size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_compact");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    if (!c) {
        set_error("ems_compact: null cache");
        return EMS_INVALID_ARGUMENT;
    }
    const ems_stage sg = st ? *st : default_stage(*d, ws);
    return run_compact(d, k_raw, v, glo, loc, sg, *c, ws, s);
}

}  // extern "C"

namespace ems {
namespace {
// The whole path on one descriptor, without resetting the status word (shared by the
// public entry points and the chunked host pipeline).
int run_path(const ems_desc* d, const void* q_rot, const void* k_rot, const void* k_raw,
             const void* v, void* out_o, float* lse, float* glo, float* loc, const ems_stage* st,
             const ems_cache& c, void* ws, cudaStream_t s, int unit_base = 0,
             cudaEvent_t o_ready = nullptr, const ScoreParts* parts = nullptr) {
    const Layout l = layout(*d);
    float* g = glo ? glo : at<float>(ws, l.glo);
    float* lc = loc ? loc : at<float>(ws, l.loc);
    const ems_stage sg = st ? *st : default_stage(*d, ws);
    if (int rc = run_score(d, q_rot, k_rot, v, out_o, lse, g, lc, ws, s, o_ready, parts)) return rc;
    if (d->seq_len > d->n_budget && d->policy != EMS_POLICY_FULL) {  // policies.cpp:136-138
        if (int rc = run_select(d, g, lc, sg, ws, s, unit_base)) return rc;
        if (int rc = run_merge(d, k_raw, v, sg, ws, s)) return rc;
    }
    return run_compact(d, k_raw, v, g, lc, sg, c, ws, s, unit_base);
}
}  // namespace
}  // namespace ems

extern "C" {

int ems_prefill_compress(const ems_desc* d, const void* q_rot, const void* k_rot,
                         const void* k_raw, const void* v, void* out_o, float* lse, float* glo,
                         float* loc, const ems_stage* st, const ems_cache* c, void* ws,
                         size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_prefill_compress");
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    if (!q_rot || !k_rot || !k_raw || !v || !c) {
        set_error("ems_prefill_compress: null tensor");
        return EMS_INVALID_ARGUMENT;
    }
    EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));
    return run_path(d, q_rot, k_rot, k_raw, v, out_o, lse, glo, loc, st, *c, ws, s);
}

int ems_rope(int32_t dtype, int32_t planes, int32_t L, int32_t d, double base, int64_t first_pos,
             const void* x, void* y, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_rope");
    if ((dtype != EMS_F32 && dtype != EMS_BF16) || planes < 0 || L < 0 || d <= 0 || d % 2 != 0 ||
        d > 512 || !(base > 0.0) || (planes > 0 && L > 0 && (!x || !y))) {
        set_error("ems_rope: bad arguments (need even head_dim <= 512, base > 0)");  // rope.cpp:11-13
        return EMS_INVALID_ARGUMENT;
    }
    if (first_pos < 0) {
        set_error("apply_rope: position must be nonnegative");  // rope.cpp:33-35
        return EMS_INVALID_ARGUMENT;
    }
    cudaError_t e = launch_rope(dtype, planes, L, d, base, first_pos, x, y, s);
    if (e != cudaSuccess) {
        set_error("rope launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int ems_prefill(const ems_desc* d, double rope_base, const void* q, const void* k, const void* v,
                void* q_rot, void* k_rot, void* out_o, float* lse, float* glo, float* loc,
                const ems_stage* st, const ems_cache* c, void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_prefill");
    if (int rc = ems_validate(d)) return rc;
    if (!(rope_base >= 0.0)) {
        set_error("ems_prefill: rope_base must be >= 0 (0 = no RoPE)");
        return EMS_INVALID_ARGUMENT;
    }
    const void* qr = q;
    const void* kr = k;
    if (rope_base > 0.0) {
        if (!q_rot || !k_rot || !q || !k) {
            set_error("ems_prefill: RoPE needs q_rot / k_rot scratch");
            return EMS_INVALID_ARGUMENT;
        }
        const int32_t pq = d->batch * d->heads_q, pk = d->batch * d->heads_kv;
        if (int rc = ems_rope(d->dtype, pq, d->seq_len, d->head_dim, rope_base, d->first_position, q,
                              q_rot, s))
            return rc;
        if (int rc = ems_rope(d->dtype, pk, d->seq_len, d->head_dim, rope_base, d->first_position, k,
                              k_rot, s))
            return rc;
        qr = q_rot;
        kr = k_rot;
    }
    return ems_prefill_compress(d, qr, kr, k, v, out_o, lse, glo, loc, st, c, ws, ws_bytes, s);
}

int ems_redundancy_cross(int32_t dtype, int32_t d, const void* k_rows, const void* v_rows,
                         int32_t n_rows, const void* k_cols, const void* v_cols, int32_t n_cols,
                         int32_t key_only, float* r, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_redundancy_cross");
    if ((dtype != EMS_F32 && dtype != EMS_BF16) || !supported_dim(d) || n_rows < 0 || n_cols < 0) {
        set_error("ems_redundancy_cross: bad arguments");
        return EMS_INVALID_ARGUMENT;
    }
    if (n_rows == 0 || n_cols == 0) return EMS_OK;
    cudaError_t e = launch_redundancy_cross(dtype, d, k_rows, v_rows, n_rows, k_cols, v_cols,
                                            n_cols, key_only, r, s);
    if (e != cudaSuccess) {
        set_error("redundancy_cross launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

size_t ems_diagnostics_workspace_bytes(int32_t units, int32_t L) {
    if (units <= 0 || L <= 0) return 0;
    return ems::diag_workspace_bytes(units, L);
}

int ems_sparsity_rate(int32_t units, int32_t L, const float* glo, const float* loc, double zeta, double* rate,
                      void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_sparsity_rate");
    using namespace ems;
    if (units <= 0 || L <= 0 || !glo || !loc || !rate || !ws) {
        set_error("ems_sparsity_rate: bad arguments");
        return EMS_INVALID_ARGUMENT;
    }
    if (!(zeta > 0.0 && zeta <= 1.0)) {  // analysis.cpp:72-74
        set_error("sparsity_rate: zeta must be in (0, 1]");
        return EMS_INVALID_ARGUMENT;
    }
    if (ws_bytes < diag_workspace_bytes(units, L)) {
        set_error("ems_sparsity_rate: workspace too small (%zu < %zu)", ws_bytes, diag_workspace_bytes(units, L));
        return EMS_INVALID_ARGUMENT;
    }
    cudaError_t e = launch_sparsity(units, L, glo, loc, zeta, rate, ws, 0, s);
    if (e != cudaSuccess) {
        set_error("sparsity launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int ems_redundancy_rate(int32_t dtype, int32_t d, int32_t units, int32_t L, const void* k, const void* v,
                        double tau, double* rate, void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_redundancy_rate");
    using namespace ems;
    if ((dtype != EMS_F32 && dtype != EMS_BF16) || !supported_dim(d) || units <= 0 || L <= 0 || !k || !v ||
        !rate || !ws) {
        set_error("ems_redundancy_rate: bad arguments");
        return EMS_INVALID_ARGUMENT;
    }
    if (ws_bytes < diag_workspace_bytes(units, L)) {
        set_error("ems_redundancy_rate: workspace too small (%zu < %zu)", ws_bytes,
                  diag_workspace_bytes(units, L));
        return EMS_INVALID_ARGUMENT;
    }
    cudaError_t e = launch_redundancy(units, L, d, dtype, k, v, tau, rate, ws, s);
    if (e != cudaSuccess) {
        set_error("redundancy launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int ems_sync_status(const ems_desc* d, void* ws, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_sync_status");
    (void)d;
    EMS_CUDA_CHECK(cudaStreamSynchronize(s));
    DevStatus st;
    EMS_CUDA_CHECK(cudaMemcpy(&st, ws, sizeof(st), cudaMemcpyDeviceToHost));
    if (st.code != 0) {
        set_error("device reported %s in unit %d", ems_status_string(st.code), st.unit);
        return st.code;
    }
    return EMS_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------------------
// Host-resident inputs: the chunked copy/compute pipeline (ems_prefill_host).
namespace ems {
namespace {

// Per-(host thread, device) pool of timing-free events and a non-blocking copy stream.
struct HostPipeRes {
    int device = -1;
    cudaStream_t copy = nullptr;
    cudaStream_t comp2 = nullptr;  // second compute stream (two unit groups in flight)
    cudaStream_t d2h = nullptr;    // device-to-host copies of the caches (the other PCIe direction)
    cudaStream_t d2h_o = nullptr;  // device-to-host copies of O (never queued behind a group's compress)
    std::vector<cudaEvent_t> ev;
};

// With two workspaces, odd groups run on a second stream with the second workspace; the
// status word of that workspace is merged into the caller's at the end.
__global__ void merge_status_kernel(DevStatus* dst, const DevStatus* src) {
    if (dst->code == 0 && src->code != 0) *dst = *src;
}
constexpr int kMaxDevices = 64;
thread_local HostPipeRes g_pipe[kMaxDevices];

HostPipeRes* pipe_res(int nev) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    HostPipeRes& r = g_pipe[dev];
    if (r.copy == nullptr && cudaStreamCreateWithFlags(&r.copy, cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    if (r.d2h == nullptr && cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    if (r.d2h_o == nullptr && cudaStreamCreateWithFlags(&r.d2h_o, cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    if (r.comp2 == nullptr && cudaStreamCreateWithFlags(&r.comp2, cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    while ((int)r.ev.size() < nev) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        r.ev.push_back(e);
    }
    r.device = dev;
    return &r;
}

template <class T>
T* off(T* p, size_t bytes) {
    return p ? reinterpret_cast<T*>(reinterpret_cast<char*>(p) + bytes) : nullptr;
}
template <class T>
const T* off(const T* p, size_t bytes) {
    return p ? reinterpret_cast<const T*>(reinterpret_cast<const char*>(p) + bytes) : nullptr;
}

// Cache arrays of units [u0, u0 + n): byte offset and size per unit of each SoA field.
struct CacheField {
    void* ems_cache::*ptr;
    size_t per_unit;
};

}  // namespace
}  // namespace ems

extern "C" int ems_prefill_host(const ems_desc* d, double rope_base, const void* h_q, const void* h_k,
                                const void* h_k_raw, const void* h_v, void* d_q, void* d_k, void* d_k_raw,
                                void* d_v, void* d_q_rot, void* d_k_rot, void* out_o, void* h_out_o, float* lse,
                                float* glo, float* loc, const ems_cache* d_cache, const ems_cache* h_cache,
                                int32_t chunks, void* ws, size_t ws_bytes, cudaStream_t s,
                                cudaStream_t copy_stream) {
    ems::NvtxRange ems_nvtx_range_("ems_prefill_host");
    using namespace ems;
    if (int rc = ems_validate(d)) return rc;
    if (int rc = check_ws(d, ws, ws_bytes)) return rc;
    const bool rope = rope_base > 0.0;
    if (!(rope_base >= 0.0) || !h_q || !h_k || !h_v || !d_q || !d_k || !d_v || !d_cache ||
        (rope && (!d_q_rot || !d_k_rot)) || (!rope && (!h_k_raw || !d_k_raw)) || (h_out_o && !out_o)) {
        set_error("ems_prefill_host: missing buffer (RoPE needs q_rot/k_rot scratch; pre-rotated "
                  "inputs need k_raw; a host O needs the device O)");
        return EMS_INVALID_ARGUMENT;
    }
    const Dims m = make_dims(*d);
    const int U = m.units, G = m.G;
    int nc = chunks < 1 ? 1 : (chunks > U ? U : chunks);
    HostPipeRes* res = pipe_res(3 * nc + 7);
    if (!res) {
        set_error("ems_prefill_host: could not create copy stream / events");
        return EMS_CUDA_ERROR;
    }
    cudaStream_t cs = copy_stream ? copy_stream : res->copy;
    // results go back on their own streams (both PCIe directions at once): caches on `ds` after
    // each group's compress, O on `dso` as soon as each group's forward pass is done
    cudaStream_t ds = res->d2h, dso = res->d2h_o;
    // [0, nc): inputs of chunk c staged; [nc, 2nc): chunk c done; [2nc, 2nc + 3): start / copies
    // done / second stream done; [2nc + 3, 3nc + 3): chunk c's O final; 3nc + 3: O copies done;
    // [3nc + 4, 3nc + 7): head parts 0 .. np-2 of chunk 0 staged (split first group)
    cudaEvent_t* ev = res->ev.data();
    cudaEvent_t* ev_o = ev + 2 * nc + 3;
    const size_t row = (size_t)m.L * m.d * m.esize;  // one [L][d] plane
    const size_t cache_d = (size_t)m.d * m.esize;
    const CacheField fields[] = {
        {(void* ems_cache::*)&ems_cache::center_key, (size_t)m.cap_c * cache_d},
        {(void* ems_cache::*)&ems_cache::center_norm, (size_t)m.cap_c * 4},
        {(void* ems_cache::*)&ems_cache::center_value, (size_t)m.cap_c * cache_d},
        {(void* ems_cache::*)&ems_cache::center_pos, (size_t)m.cap_c * 4},
        {(void* ems_cache::*)&ems_cache::center_score, (size_t)m.cap_c * 12},
        {(void* ems_cache::*)&ems_cache::local_key, (size_t)m.cap_l * cache_d},
        {(void* ems_cache::*)&ems_cache::local_value, (size_t)m.cap_l * cache_d},
        {(void* ems_cache::*)&ems_cache::local_pos, (size_t)m.cap_l * 4},
        {(void* ems_cache::*)&ems_cache::local_score, (size_t)m.cap_l * 12},
        {(void* ems_cache::*)&ems_cache::lut_pos, (size_t)(m.cap_lut > 0 ? m.cap_lut : 1) * 4},
        {(void* ems_cache::*)&ems_cache::lut_slot, (size_t)(m.cap_lut > 0 ? m.cap_lut : 1) * 4},
        {(void* ems_cache::*)&ems_cache::counts, 16},
    };
    // two unit groups in flight (odd groups on a second stream and workspace) when the caller
    // passed ems_prefill_host_workspace_bytes(); one at a time otherwise
    const size_t one = align_up(workspace_need(*d));
    // RoPE (cos, sin) computed once for every group when the workspace has room for the table
    const size_t tab_bytes = align_up(rope_table64_bytes(m.L, m.d));
    const bool dual = nc >= 2 && ws_bytes >= 2 * one;
    const bool use_tab = rope && ws_bytes >= (dual ? 2 : 1) * one + tab_bytes;
    void* ws2 = dual ? off(ws, one) : nullptr;
    void* tab = use_tab ? off(ws, (dual ? 2 : 1) * one) : nullptr;
    cudaStream_t s2 = dual ? res->comp2 : s;
    // Everything below is stream-ordered.  Whatever happens (a failed launch part-way through the
    // groups included), `stream` is finally ordered after the copy stream and the second compute
    // stream, so a caller that synchronises it never races with copies still in flight.
    const int rc = [&]() -> int {
        EMS_CUDA_CHECK(cudaMemsetAsync(ws, 0, sizeof(DevStatus), s));
        if (dual) EMS_CUDA_CHECK(cudaMemsetAsync(ws2, 0, sizeof(DevStatus), s));
        // the copy stream (and the second compute stream) must not overwrite device inputs that
        // earlier work on `s` still reads
        EMS_CUDA_CHECK(cudaEventRecord(ev[2 * nc], s));
        EMS_CUDA_CHECK(cudaStreamWaitEvent(cs, ev[2 * nc], 0));
        if (dual) EMS_CUDA_CHECK(cudaStreamWaitEvent(s2, ev[2 * nc], 0));
        // Geometric groups (U / 2^(nc-1), ..., U / 4, U / 2 units): the first group's inputs land
        // after a small copy, so compute starts early; later groups are large (efficient grids)
        // and their copies finish while earlier groups compute.
        auto group_end = [&](int c) {
            if (c >= nc - 1) return U;
            const long long e = ((long long)U + (1ll << (nc - 1 - c)) - 1) >> (nc - 1 - c);
            return (int)(e < c + 1 ? c + 1 : e);
        };
        auto unit_range = [&](int c, int& u0, int& n) {
            u0 = c == 0 ? 0 : group_end(c - 1);
            n = group_end(c) - u0;
        };
        // The first group's forward pass runs in two halves of the query heads, each as soon as K,
        // V and its heads' Q have landed: the pipeline fill shrinks from G + 2 to G / 2 + 2 head
        // planes per unit (config 3: 50 -> 34 MB) and the second half's copy runs under the first
        // half's compute (four one-head parts were slower: 128-pair launches leave most of the last
        // wave idle)
        const int np = nc >= 2 && G >= 2 && G % 2 == 0 ? 2 : 1;
        const bool split0 = np > 1;
        const int hp = G / np;  // heads per part
        const cudaEvent_t* ev_part = ev + 3 * nc + 4;
        // (1) H2D of every chunk, in chunk order (score inputs first, the raw K of a pre-rotated
        //     problem last since only the merge/compact stages read it)
        for (int c = 0; c < nc; ++c) {
            int u0, n;
            unit_range(c, u0, n);
            const size_t oq = (size_t)u0 * G * row, nq = (size_t)n * G * row;
            const size_t ok = (size_t)u0 * row, nk = (size_t)n * row;
            if (c == 0 && split0) {  // K, V, then each unit's heads part by part
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_k, ok), off(h_k, ok), nk, cudaMemcpyHostToDevice, cs));
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_v, ok), off(h_v, ok), nk, cudaMemcpyHostToDevice, cs));
                for (int pt = 0; pt < np; ++pt) {
                    for (int u = 0; u < n; ++u) {
                        const size_t o = oq + ((size_t)u * G + pt * hp) * row;
                        EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_q, o), off(h_q, o), (size_t)hp * row,
                                                       cudaMemcpyHostToDevice, cs));
                    }
                    if (pt < np - 1) EMS_CUDA_CHECK(cudaEventRecord(ev_part[pt], cs));
                }
            } else {
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_q, oq), off(h_q, oq), nq, cudaMemcpyHostToDevice, cs));
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_k, ok), off(h_k, ok), nk, cudaMemcpyHostToDevice, cs));
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_v, ok), off(h_v, ok), nk, cudaMemcpyHostToDevice, cs));
            }
            if (!rope)
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(d_k_raw, ok), off(h_k_raw, ok), nk, cudaMemcpyHostToDevice, cs));
            EMS_CUDA_CHECK(cudaEventRecord(ev[c], cs));
        }
        // the RoPE table, enqueued after the copies so that they start first; it runs under the
        // first group's copies, and the second compute stream waits for it too
        if (use_tab) {
            EMS_CUDA_CHECK(launch_rope_table64(tab, m.L, m.d, rope_base, d->first_position, s));
            EMS_CUDA_CHECK(cudaEventRecord(ev[2 * nc + 2], s));
            if (dual) EMS_CUDA_CHECK(cudaStreamWaitEvent(s2, ev[2 * nc + 2], 0));
        }
        // (2) compute chunk c once its inputs landed; (3) copy its cache back as soon as it is done
        for (int c = 0; c < nc; ++c) {
            int u0, n;
            unit_range(c, u0, n);
            ems_desc sub = *d;
            sub.batch = 1;
            sub.heads_kv = n;
            sub.heads_q = n * G;
            const size_t oq = (size_t)u0 * G * row, ok = (size_t)u0 * row;
            cudaStream_t sc = (c & 1) ? s2 : s;
            void* wsc = dual && (c & 1) ? ws2 : ws;
            const bool split = c == 0 && split0;
            EMS_CUDA_CHECK(cudaStreamWaitEvent(sc, split ? ev_part[0] : ev[c], 0));
            const void* qr = off(d_q, oq);
            const void* kr = off(d_k, ok);
            const void* kraw = rope ? kr : off(d_k_raw, ok);
            auto rope_planes = [&](int planes, const void* x, void* y) -> cudaError_t {
                return use_tab ? launch_rope_tab(d->dtype, planes, m.L, m.d, tab, x, y, sc)
                               : launch_rope(d->dtype, planes, m.L, m.d, rope_base, d->first_position, x, y, sc);
            };
            // RoPE of query heads [h0, h0 + nh) of every unit of the group
            auto rope_q = [&](int h0, int nh) -> cudaError_t {
                if (nh == G) return rope_planes(n * G, off(d_q, oq), off(d_q_rot, oq));
                for (int u = 0; u < n; ++u) {
                    const size_t o = oq + ((size_t)u * G + h0) * row;
                    cudaError_t e = rope_planes(nh, off(d_q, o), off(d_q_rot, o));
                    if (e != cudaSuccess) return e;
                }
                return cudaSuccess;
            };
            if (rope) {
                if (!split) EMS_CUDA_CHECK(rope_q(0, G));
                EMS_CUDA_CHECK(rope_planes(n, kr, off(d_k_rot, ok)));
                qr = off(d_q_rot, oq);
                kr = off(d_k_rot, ok);
            }
            ScoreParts parts;
            if (split) {
                parts.n = np;
                parts.before = [&](int part, cudaStream_t st) -> cudaError_t {
                    if (part > 0) {  // this part's heads (the last part: every input of the group)
                        cudaError_t e = cudaStreamWaitEvent(st, part < np - 1 ? ev_part[part] : ev[0], 0);
                        if (e != cudaSuccess) return e;
                    }
                    return rope ? rope_q(part * hp, hp) : cudaSuccess;
                };
            }
            ems_cache scache = *d_cache;
            for (const CacheField& f : fields) scache.*f.ptr = off(d_cache->*f.ptr, (size_t)u0 * f.per_unit);
            const size_t ol = (size_t)u0 * m.L;
            if (int rc = run_path(&sub, qr, kr, kraw, off(d_v, ok), off(out_o, oq), off(lse, (size_t)u0 * G * m.L * 4),
                                  off(glo, ol * 4), off(loc, ol * 4), nullptr, scache, wsc, sc, u0,
                                  h_out_o ? ev_o[c] : nullptr, split ? &parts : nullptr))
                return rc;
            EMS_CUDA_CHECK(cudaEventRecord(ev[nc + c], sc));
            if (h_out_o) {  // engine::prefill's PrefillResult.per_head outputs (engine.hpp:36-45): O is final
                            // after the forward pass, so its copy overlaps this group's column sums and compress
                EMS_CUDA_CHECK(cudaStreamWaitEvent(dso, ev_o[c], 0));
                // ... and after the next group's inputs landed: concurrent D2H slows the host-to-device
                // copies the next group waits for (measured 55 -> 32 GB/s), O has slack
                if (c + 1 < nc) EMS_CUDA_CHECK(cudaStreamWaitEvent(dso, ev[c + 1], 0));
                EMS_CUDA_CHECK(cudaMemcpyAsync(off(h_out_o, oq), off(out_o, oq), (size_t)n * G * row,
                                               cudaMemcpyDeviceToHost, dso));
            }
            if (h_cache) {
                EMS_CUDA_CHECK(cudaStreamWaitEvent(ds, ev[nc + c], 0));
                for (const CacheField& f : fields)
                    EMS_CUDA_CHECK(cudaMemcpyAsync(off(h_cache->*f.ptr, (size_t)u0 * f.per_unit), scache.*f.ptr,
                                                   (size_t)n * f.per_unit, cudaMemcpyDeviceToHost, ds));
            }
        }
        return EMS_OK;
    }();
    cudaEventRecord(ev[2 * nc + 1], cs);
    cudaStreamWaitEvent(s, ev[2 * nc + 1], 0);
    cudaEventRecord(ev[2 * nc], ds);  // the start event's slot is free again: reuse it for the D2H stream
    cudaStreamWaitEvent(s, ev[2 * nc], 0);
    cudaEventRecord(ev[3 * nc + 3], dso);
    cudaStreamWaitEvent(s, ev[3 * nc + 3], 0);
    if (dual) {
        cudaEventRecord(ev[2 * nc + 2], s2);
        cudaStreamWaitEvent(s, ev[2 * nc + 2], 0);
        if (rc == EMS_OK) {
            merge_status_kernel<<<1, 1, 0, s>>>(static_cast<DevStatus*>(ws), static_cast<const DevStatus*>(ws2));
            EMS_CUDA_CHECK(cudaGetLastError());
        }
    }
    return rc;
}

// ----------------------------------------------------------------------------------------
// Decode (decode_step / decode_update).
namespace ems {
namespace {
// Per-unit capacities.  EMS / H2O / StreamingLLM keep the centers at capacity (one extra
// slot for the graduating token); SnapKV and full let decode tokens accumulate
// (policies.cpp:186-191), so they are sized by the decode horizon max_pos - seq_len.
void decode_caps(const ems_desc& d, int max_pos, int& S, int& W, int& T, int& R) {
    const Dims m = make_dims(d);
    const int steps = max_pos > d.seq_len ? max_pos - d.seq_len : 0;
    const int wl = (d.l_win > d.n_budget ? d.l_win : d.n_budget) + 1;
    switch (d.policy) {
        case EMS_POLICY_FULL:
            S = 1;
            W = (d.seq_len > d.n_budget ? d.seq_len : d.n_budget) + steps + 1;
            T = 1;
            break;
        case EMS_POLICY_SNAPKV:
            S = m.cap_c + steps + 1;
            W = wl;
            T = S;
            break;
        case EMS_POLICY_H2O:
        case EMS_POLICY_STREAMING:
            S = m.cap_c + 1;
            W = wl;
            T = S;
            break;
        default:
            S = m.cap_c + 1;
            W = wl;
            T = (int)(d.gamma * (double)d.n_budget);  // lut_capacity, cache.hpp:36-38
            if (T < m.cap_lut) T = m.cap_lut;
    }
    R = T + W;
}
int decode_check(const ems_desc* d, int max_pos) {
    if (int rc = ems_validate(d)) return rc;
    if (d->heads_q / d->heads_kv > 8) {
        set_error("decode: at most 8 query heads per KV head");
        return EMS_UNSUPPORTED;
    }
    if (d->position_mode != 0 && d->position_mode != 1) {
        set_error("bad position_mode");
        return EMS_INVALID_ARGUMENT;
    }
    if (max_pos < d->seq_len) {
        set_error("decode: max_positions %d < seq_len %d", max_pos, d->seq_len);
        return EMS_INVALID_ARGUMENT;
    }
    // the step keeps one fp64 accumulator per slot + local in shared memory: the full and SnapKV
    // policies grow S + W with the prompt and the horizon
    int S, W, T, R;
    decode_caps(*d, max_pos, S, W, T, R);
    const size_t smem = decode_smem_bytes(make_dims(*d), S, W);
    constexpr size_t kSmemLimit = 227 * 1024 - 8 * 1024;  // opt-in maximum minus the static part
    if (smem > kSmemLimit) {
        set_error("decode: %zu B of shared memory for %d slots + %d locals exceeds the %zu B available "
                  "(shorter prompt or horizon, or the EMS / H2O / StreamingLLM policies)",
                  smem, S, W, kSmemLimit);
        return EMS_UNSUPPORTED;
    }
    return EMS_OK;
}
}  // namespace
}  // namespace ems

extern "C" {

int ems_decode_dims_for(const ems_desc* d, int32_t max_pos, ems_decode_dims* out) {
    using namespace ems;
    if (int rc = decode_check(d, max_pos)) return rc;
    int S, W, T, R;
    decode_caps(*d, max_pos, S, W, T, R);
    out->units = d->batch * d->heads_kv;
    out->slots = S;
    out->locals = W;
    out->lut = T;
    out->rows = R;
    return EMS_OK;
}

size_t ems_decode_workspace_bytes(const ems_desc* d, int32_t max_pos) {
    using namespace ems;
    if (decode_check(d, max_pos) != EMS_OK) return 0;
    int S, W, T, R;
    decode_caps(*d, max_pos, S, W, T, R);
    return decode_workspace_bytes(make_dims(*d), R);
}

int ems_rope_table(int32_t d, double base, int32_t max_pos, void* table, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_rope_table");
    using namespace ems;
    if (d <= 0 || d % 2 || !(base > 0.0) || max_pos <= 0 || !table) {
        set_error("ems_rope_table: bad arguments");
        return EMS_INVALID_ARGUMENT;
    }
    cudaError_t e = launch_rope_table(static_cast<float2*>(table), max_pos, d, base, s);
    if (e != cudaSuccess) {
        set_error("rope table launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int ems_decode_init(const ems_desc* d, int32_t max_pos, const ems_cache* c, const ems_decode_state* st,
                    cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_decode_init");
    using namespace ems;
    if (int rc = decode_check(d, max_pos)) return rc;
    if (!c || !st) {
        set_error("ems_decode_init: null cache/state");
        return EMS_INVALID_ARGUMENT;
    }
    int S, W, T, R;
    decode_caps(*d, max_pos, S, W, T, R);
    cudaError_t e = launch_decode_init(make_dims(*d), d->dtype, *c, *st, S, W, T, s);
    if (e != cudaSuccess) {
        set_error("decode init launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

int ems_decode_sync_status(const ems_desc* d, const ems_decode_state* st, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_decode_sync_status");
    using namespace ems;
    if (int rc = ems_validate(d)) return rc;
    if (!st || !st->meta) {
        set_error("ems_decode_sync_status: null state");
        return EMS_INVALID_ARGUMENT;
    }
    const int U = d->batch * d->heads_kv;
    std::vector<int32_t> meta((size_t)U * 8);
    EMS_CUDA_CHECK(cudaStreamSynchronize(s));
    EMS_CUDA_CHECK(cudaMemcpy(meta.data(), st->meta, meta.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int u = 0; u < U; ++u)
        if (meta[(size_t)u * 8 + 6] != 0) {
            set_error("decode state of unit %d is corrupt (stepped past its capacity or no free slot)", u);
            return meta[(size_t)u * 8 + 6];
        }
    return EMS_OK;
}

int ems_decode_step(const ems_desc* d, int64_t position, const void* table, int32_t max_pos, const void* q,
                    const void* k, const void* v, void* out, int32_t* argmax_pos, const ems_decode_state* st,
                    void* ws, size_t ws_bytes, cudaStream_t s) {
    ems::NvtxRange ems_nvtx_range_("ems_decode_step");
    using namespace ems;
    if (int rc = decode_check(d, max_pos)) return rc;
    if (!table || !q || !k || !v || !out || !argmax_pos || !st) {
        set_error("ems_decode_step: null argument");
        return EMS_INVALID_ARGUMENT;
    }
    if (position < 0 || position >= max_pos) {
        set_error("ems_decode_step: position %lld outside the RoPE table [0, %d)", (long long)position, max_pos);
        return EMS_INVALID_ARGUMENT;
    }
    int S, W, T, R;
    decode_caps(*d, max_pos, S, W, T, R);
    const Dims m = make_dims(*d);
    if (!ws || ws_bytes < decode_workspace_bytes(m, R)) {
        set_error("ems_decode_step: workspace too small (need %zu)", decode_workspace_bytes(m, R));
        return EMS_INVALID_ARGUMENT;
    }
    cudaError_t e = launch_decode_step(m, d->dtype, S, W, T, R, d->l_win, T, d->tau, d->zero_class,
                                       d->position_mode == 0, position, max_pos, static_cast<const float2*>(table),
                                       q, k, v, out, argmax_pos, *st, ws, s, d->policy, d->sink_count,
                                       d->n_budget);
    if (e != cudaSuccess) {
        set_error("decode step launch: %s", cudaGetErrorString(e));
        return EMS_CUDA_ERROR;
    }
    return EMS_OK;
}

}  // extern "C"
