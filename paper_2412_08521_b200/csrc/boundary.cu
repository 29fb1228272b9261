// boundary.cu -- the reference's fine-grained operator entry points as stand-alone device
// kernels, so a caller of proj/include/ems/{scoring,compressor}.hpp can swap every function of
// the prefill path, not only the fused pipeline (include/ems_b200/ems.hpp binds them):
//
//   effective_score            scoring.cpp:146-152 (+ combine_glo_loc :105-124, mean_pool_1d
//                              numerics.cpp:62-82)                       -> effective_score_kernel
//   partition_tokens           compressor.cpp:48-74   -> the select kernels on caller scores
//                              (select.cu, kPolicyPooled; launched from capi.cu)
//   assign_merge_destinations  compressor.cpp:76-95                      -> assign_rows_kernel
//   weighted_merge             compressor.cpp:97-161                     -> weighted_merge_kernel
//
// The fused hot path (ems_prefill_compress) never calls these; they exist for API parity.
#include "common.cuh"

namespace ems {

namespace {

constexpr int kEffThreads = 1024;

__device__ double block_sum_d(double v, double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];  // fixed order: deterministic
    __syncthreads();
    return t;
}

// mean_pool_1d(combine_glo_loc(glo, loc_past + loc_cur), kernel) per unit, fp64 arithmetic on the
// fp32 device scores (contract D9), one CTA per unit.  Zero global mass records
// EMS_DEGENERATE_INPUT (DegenerateInputError, scoring.cpp:115-117) and writes zeros.
__global__ void __launch_bounds__(kEffThreads) effective_score_kernel(const float* __restrict__ glo,
                                                                      const float* __restrict__ loc_past,
                                                                      const float* __restrict__ loc_cur, int L,
                                                                      int kernel, float* __restrict__ pooled,
                                                                      DevStatus* status) {
    __shared__ double sh[32];
    const int u = blockIdx.x, tid = threadIdx.x;
    const float* g = glo + (size_t)u * L;
    const float* lp = loc_past + (size_t)u * L;
    const float* lc = loc_cur ? loc_cur + (size_t)u * L : nullptr;
    float* out = pooled + (size_t)u * L;
    auto loc_at = [&](int i) { return (double)lp[i] + (lc ? (double)lc[i] : 0.0); };
    double sg = 0.0, sl = 0.0;
    for (int i = tid; i < L; i += kEffThreads) sg += (double)g[i], sl += loc_at(i);
    sg = block_sum_d(sg, sh);
    sl = block_sum_d(sl, sh);
    if (!(sg > 0.0)) {
        if (tid == 0) record_status(status, EMS_DEGENERATE_INPUT, u);
        for (int i = tid; i < L; i += kEffThreads) out[i] = 0.f;
        return;
    }
    const double align = sl / sg;
    const int half = kernel / 2;
    for (int i = tid; i < L; i += kEffThreads) {
        const int a = max(0, i - half), b = min(L - 1, i + half);
        double acc = 0.0;
        for (int j = a; j <= b; ++j) {
            const double x = (double)g[j] * align, y = loc_at(j);
            acc += x > y ? x : y;
        }
        out[i] = (float)(acc / (double)(b - a + 1));
    }
}

// Row argmax with the reference's strict '>' (ties -> lower column), then the tau threshold.
__global__ void __launch_bounds__(256) assign_rows_kernel(const float* __restrict__ r, int n_rows, int n_cols,
                                                          double tau, int32_t* __restrict__ dest) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= n_rows) return;
    float best = -INFINITY;
    int best_c = n_cols;  // sentinel: larger than any column
    for (int c = lane; c < n_cols; c += 32) {
        const float x = r[(size_t)row * n_cols + c];
        if (best_c == n_cols || x > best) best = x, best_c = c;  // per lane: ascending columns
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
        if (oc < n_cols && (best_c == n_cols || ob > best || (ob == best && oc < best_c))) best = ob, best_c = oc;
    }
    if (lane == 0) dest[row] = (best_c < n_cols && (double)best >= tau) ? best_c : -1;
}

// weighted_merge: one warp per center column.  Members are the TBM rows whose destination is the
// column, in ascending row order (the reference's member order), found by one ordered pass over
// the destinations; all arithmetic in fp64 as the reference's.
__global__ void __launch_bounds__(256) weighted_merge_kernel(
    int d, int n_cols, double* __restrict__ center_unit_key, double* __restrict__ center_value,
    double* __restrict__ center_score, const double* __restrict__ center_weight, int n_tbm,
    const double* __restrict__ tbm_key, const double* __restrict__ tbm_value, const double* __restrict__ tbm_weight,
    const double* __restrict__ tbm_score, const int32_t* __restrict__ dest) {
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (c >= n_cols) return;
    double ws = center_weight[c];
    int members = 0;
    for (int i = 0; i < n_tbm; ++i)
        if (dest[i] == c) ws += tbm_weight[i], ++members;
    if (members == 0) return;
    const double uniform = 1.0 / (double)(members + 1);
    double* uk = center_unit_key + (size_t)c * d;
    double* val = center_value + (size_t)c * d;
    const double wc = ws > 0.0 ? center_weight[c] / ws : uniform;
    constexpr int kMaxR = 16;  // d <= 512
    double mk[kMaxR], mv[kMaxR];
    for (int r = 0; r < kMaxR; ++r) {
        const int x = lane + 32 * r;
        mk[r] = x < d ? wc * uk[x] : 0.0;
        mv[r] = x < d ? wc * val[x] : 0.0;
    }
    double s0 = center_score[3 * c], s1 = center_score[3 * c + 1], s2 = center_score[3 * c + 2];
    for (int i = 0; i < n_tbm; ++i) {
        if (dest[i] != c) continue;
        const double* kr = tbm_key + (size_t)i * d;
        double ss = 0.0;
        for (int x = lane; x < d; x += 32) ss += kr[x] * kr[x];
        ss = warp_sum(ss);
        const double nrm = sqrt(ss);  // normalized_or_zero, compressor.cpp:16-25
        const double w = ws > 0.0 ? tbm_weight[i] / ws : uniform;
        for (int r = 0; r < kMaxR; ++r) {
            const int x = lane + 32 * r;
            if (x < d) {
                mk[r] += w * (nrm > 0.0 ? kr[x] / nrm : 0.0);
                mv[r] += w * tbm_value[(size_t)i * d + x];
            }
        }
        s0 += tbm_score[3 * i];
        s1 += tbm_score[3 * i + 1];
        s2 += tbm_score[3 * i + 2];
    }
    double ss = 0.0;
    for (int r = 0; r < kMaxR; ++r) ss += mk[r] * mk[r];
    const double mn = sqrt(warp_sum(ss));
    for (int r = 0; r < kMaxR; ++r) {
        const int x = lane + 32 * r;
        if (x < d) {
            if (mn > 0.0) uk[x] = mk[r] / mn;  // a zero merged key keeps the center's unit key
            val[x] = mv[r];
        }
    }
    if (lane == 0) center_score[3 * c] = s0, center_score[3 * c + 1] = s1, center_score[3 * c + 2] = s2;
}

}  // namespace

cudaError_t launch_effective_score(int units, int L, int kernel, const float* glo, const float* loc_past,
                                   const float* loc_cur, float* pooled, DevStatus* status, cudaStream_t s) {
    effective_score_kernel<<<units, kEffThreads, 0, s>>>(glo, loc_past, loc_cur, L, kernel, pooled, status);
    return cudaGetLastError();
}

cudaError_t launch_assign_rows(const float* r, int n_rows, int n_cols, double tau, int32_t* dest, cudaStream_t s) {
    if (n_rows > 0) assign_rows_kernel<<<(n_rows + 7) / 8, 256, 0, s>>>(r, n_rows, n_cols, tau, dest);
    return cudaGetLastError();
}

cudaError_t launch_weighted_merge(int d, int n_cols, double* uk, double* val, double* score, const double* cw,
                                  int n_tbm, const double* tk, const double* tv, const double* tw, const double* ts,
                                  const int32_t* dest, cudaStream_t s) {
    if (n_cols > 0)
        weighted_merge_kernel<<<(n_cols + 7) / 8, 256, 0, s>>>(d, n_cols, uk, val, score, cw, n_tbm, tk, tv, tw, ts,
                                                               dest);
    return cudaGetLastError();
}

}  // namespace ems
