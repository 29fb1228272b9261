// score_simt.cu -- SIMT (FFMA) score pass: causal attention O + row LSE, then
// deterministic GQA-mean column sums (glo, loc).
//
// Used for fp32 inputs (config 1: tcgen05 has no fp32-input MMA kind that keeps
// the 1e-4 contract) and as the independent second GPU
// implementation the tcgen05 kernels are cross-checked against.
//
// Reference semantics: streaming_pass, proj/src/scoring.cpp:20-64 --
//   P_ij = softmax_j(q_i . k_j / sqrt(d)) over j <= i,   O_i = sum_j P_ij v_j,
//   glo_j = sum_{i >= j} P_ij,  loc_j = sum_{i >= L - w} P_ij   (w = min(l_win, L)).
// GQA (contract D2): unit scores are the mean over the unit's G query heads.
#include "common.cuh"

namespace ems {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// One warp per query row; keys streamed 32 at a time (one per lane), online
// softmax in the exp2 domain, O accumulated with lane-owned dimensions.
template <typename T, int D>
__global__ void __launch_bounds__(256) fwd_simt_kernel(const T* __restrict__ q,
                                                       const T* __restrict__ k,
                                                       const T* __restrict__ v, T* __restrict__ o,
                                                       float* __restrict__ lse, int Hq, int Hkv,
                                                       int G, int L, float qscale) {
    constexpr int R = (D + 31) / 32;  // dims per lane (lanes >= D idle when D < 32)
    __shared__ float qs[8][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * 8 + warp;
    const int bh = blockIdx.y;
    const int b = bh / Hq, hq = bh % Hq, hk = hq / G;
    if (row >= L) return;
    const T* qr = q + ((size_t)bh * L + row) * D;
    const T* kb = k + ((size_t)(b * Hkv + hk) * L) * D;
    const T* vb = v ? v + ((size_t)(b * Hkv + hk) * L) * D : nullptr;
    for (int x = lane; x < D; x += 32) qs[warp][x] = ld(qr + x) * qscale;
    __syncwarp();
    float m = -INFINITY, l = 0.f;
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    for (int j0 = 0; j0 <= row; j0 += 32) {
        const int j = j0 + lane;
        float s = -INFINITY;
        if (j <= row) {
            const T* kr = kb + (size_t)j * D;
            float a = 0.f;
#pragma unroll 8
            for (int x = 0; x < D; ++x) a = fmaf(qs[warp][x], ld(kr + x), a);
            s = a;
        }
        const float mn = fmaxf(m, warp_max(s));
        const float p = (j <= row) ? exp2f(s - mn) : 0.f;
        const float corr = exp2f(m - mn);  // m = -inf on the first chunk -> 0
        l = l * corr + warp_sum(p);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] *= corr;
        m = mn;
        if (vb) {
            const int nj = min(32, row - j0 + 1);
            for (int t = 0; t < nj; ++t) {
                const float pt = __shfl_sync(0xffffffffu, p, t);
                const T* vr = vb + (size_t)(j0 + t) * D;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (lane + 32 * r < D) acc[r] = fmaf(pt, ld(vr + lane + 32 * r), acc[r]);
            }
        }
    }
    if (o) {
        T* orow = o + ((size_t)bh * L + row) * D;
        const float inv = 1.f / l;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (lane + 32 * r < D) st(orow + lane + 32 * r, acc[r] * inv);
    }
    if (lse && lane == 0) lse[(size_t)bh * L + row] = (m + log2f(l)) * kLn2;
}

// Column sums.  Block = 32 keys (one per lane) x 8 warps splitting the query
// rows; per-lane fp64 accumulation, then a fixed-order cross-warp reduction,
// so the result is deterministic.  lse is the natural-log row LSE from above.
template <typename T, int D>
__global__ void __launch_bounds__(256) colsum_simt_kernel(const T* __restrict__ q,
                                                          const T* __restrict__ k,
                                                          const float* __restrict__ lse,
                                                          float* __restrict__ glo,
                                                          float* __restrict__ loc, int Hq, int Hkv,
                                                          int G, int L, int lwin, float qscale) {
    __shared__ float ks[D][33];
    __shared__ float qs[8][D];
    __shared__ double red[2][8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * 32;
    const int unit = blockIdx.y;
    const int b = unit / Hkv, hk = unit % Hkv;
    const T* kb = k + ((size_t)unit * L) * D;
    for (int e = threadIdx.x; e < 32 * D; e += 256) {
        const int jj = e / D, x = e % D;
        ks[x][jj] = (j0 + jj < L) ? ld(kb + (size_t)(j0 + jj) * D + x) : 0.f;
    }
    __syncthreads();
    const int j = j0 + lane;
    const int loc_start = L - lwin;
    double ag = 0.0, al = 0.0;
    for (int h = 0; h < G; ++h) {
        const int hq = hk * G + h;
        const size_t bh = (size_t)b * Hq + hq;
        const T* qb = q + bh * L * D;
        const float* lb = lse + bh * L;
        for (int i = j0 + warp; i < L; i += 8) {
            __syncwarp();
            for (int x = lane; x < D; x += 32) qs[warp][x] = ld(qb + (size_t)i * D + x) * qscale;
            __syncwarp();
            float s = 0.f;
#pragma unroll 8
            for (int x = 0; x < D; ++x) s = fmaf(qs[warp][x], ks[x][lane], s);
            const float p = (i >= j && j < L) ? exp2f(s - lb[i] * kLog2e) : 0.f;
            ag += p;
            if (i >= loc_start) al += p;
        }
    }
    red[0][warp][lane] = ag;
    red[1][warp][lane] = al;
    __syncthreads();
    if (warp == 0 && j < L) {
        double sg = 0.0, sl = 0.0;
        for (int w = 0; w < 8; ++w) sg += red[0][w][lane], sl += red[1][w][lane];
        glo[(size_t)unit * L + j] = (float)(sg / G);
        loc[(size_t)unit * L + j] = (float)(sl / G);
    }
}

template <typename T, int D>
cudaError_t launch_simt(const Dims& dm, const void* q, const void* k, const void* v, void* o,
                        float* lse, float* glo, float* loc, cudaStream_t s) {
    const float qscale = kLog2e / sqrtf((float)dm.d);
    dim3 g1((dm.L + 7) / 8, dm.B * dm.Hq);
    fwd_simt_kernel<T, D><<<g1, 256, 0, s>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, lse,
                                            dm.Hq, dm.Hkv, dm.G, dm.L, qscale);
    dim3 g2((dm.L + 31) / 32, dm.units);
    colsum_simt_kernel<T, D><<<g2, 256, 0, s>>>((const T*)q, (const T*)k, lse, glo, loc, dm.Hq,
                                               dm.Hkv, dm.G, dm.L, dm.lwin_scores, qscale);
    return cudaGetLastError();
}

}  // namespace

// lse is required here (the column pass normalises with it); the caller passes
// a workspace buffer when the user did not ask for it.
cudaError_t score_simt(const Dims& dm, int dtype, const void* q, const void* k, const void* v,
                       void* o, float* lse, float* glo, float* loc, cudaStream_t s) {
#define EMS_SIMT_CASE(T, D) \
    if (dm.d == D) return launch_simt<T, D>(dm, q, k, v, o, lse, glo, loc, s);
    if (dtype == EMS_F32) {
        EMS_SIMT_CASE(float, 8)
        EMS_SIMT_CASE(float, 16)
        EMS_SIMT_CASE(float, 32)
        EMS_SIMT_CASE(float, 64)
        EMS_SIMT_CASE(float, 96)
        EMS_SIMT_CASE(float, 128)
    } else {
        EMS_SIMT_CASE(__nv_bfloat16, 8)
        EMS_SIMT_CASE(__nv_bfloat16, 16)
        EMS_SIMT_CASE(__nv_bfloat16, 32)
        EMS_SIMT_CASE(__nv_bfloat16, 64)
        EMS_SIMT_CASE(__nv_bfloat16, 96)
        EMS_SIMT_CASE(__nv_bfloat16, 128)
    }
#undef EMS_SIMT_CASE
    return cudaErrorInvalidValue;
}

}  // namespace ems
