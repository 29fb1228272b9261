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

// Tiled FFMA kernels: a block owns 64 query rows (forward) or 64 keys (column sums) and streams
// 64-row tiles of the other operand through shared memory; 256 threads as 16 x 16, thread (ty, tx)
// holding a 4 x 4 block of the score tile (rows 4 ty + i, columns tx + 16 j).  Row / column
// reductions go across the 16 threads of a half-warp in a fixed shuffle order, and per-tile fp32
// partial sums enter fp64 accumulators in tile order, so results are deterministic.
constexpr int kBM = 64;      // rows per tile (queries in the forward, keys in the column sums)
constexpr int kBN = 64;      // columns per tile
constexpr int kST = 256;     // threads

template <int D>
struct SimtSmem {
    static constexpr int kLd = D + 1;                                   // padded row stride (banks)
    static constexpr size_t kFwd = sizeof(float) * (2 * kBM * kLd + kBN * D + kBM * (kBN + 1));
    static constexpr size_t kCol = sizeof(float) * (2 * kBM * kLd + kBN);
};

__device__ __forceinline__ float hmax16(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float hsum16(float v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double hsum16(double v) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// rows [r0, r0 + 64) of a [L][D] plane into s[64][D + 1] (fp32, scaled), zero past L
template <typename T, int D>
__device__ __forceinline__ void load_tile(float* s, const T* __restrict__ src, int r0, int L, float scale) {
    for (int e = threadIdx.x; e < kBM * D; e += kST) {
        const int r = e / D, x = e % D;
        s[r * (D + 1) + x] = (r0 + r < L) ? ld(src + (size_t)(r0 + r) * D + x) * scale : 0.f;
    }
}

// Forward: O and the row LSE, online softmax in the exp2 domain.  grid (ceil(L/64), B*Hq).
template <typename T, int D>
__global__ void __launch_bounds__(kST) fwd_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                       const T* __restrict__ v, T* __restrict__ o,
                                                       float* __restrict__ lse, int Hq, int Hkv, int G, int L,
                                                       float qscale) {
    constexpr int LD = D + 1, DC = (D + 15) / 16;
    extern __shared__ float sm[];
    float* Qs = sm;                   // [64][D+1] scaled by log2(e)/sqrt(d)
    float* Ks = Qs + kBM * LD;        // [64][D+1]
    float* Vs = Ks + kBN * LD;        // [64][D]
    float* Ps = Vs + kBN * D;         // [64][65]
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int r0 = blockIdx.x * kBM, bh = blockIdx.y;
    const int b = bh / Hq, hq = bh % Hq, hk = hq / G;
    const T* kb = k + (size_t)(b * Hkv + hk) * L * D;
    const T* vb = v ? v + (size_t)(b * Hkv + hk) * L * D : nullptr;
    load_tile<T, D>(Qs, q + (size_t)bh * L * D, r0, L, qscale);
    float m[4], l[4], acc[4][DC];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int c = 0; c < DC; ++c) acc[i][c] = 0.f;
    }
    const int last_row = min(L, r0 + kBM) - 1;
    for (int j0 = 0; j0 <= last_row; j0 += kBN) {
        __syncthreads();  // previous tile's Ks / Vs / Ps reads done
        load_tile<T, D>(Ks, kb, j0, L, 1.f);
        if (vb)
            for (int e = tid; e < kBN * D; e += kST) {
                const int r = e / D, x = e % D;
                Vs[e] = (j0 + r < L) ? ld(vb + (size_t)(j0 + r) * D + x) : 0.f;
            }
        __syncthreads();
        float sc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) sc[i][j] = 0.f;
#pragma unroll 4
        for (int x = 0; x < D; ++x) {
            float qv[4], kv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) qv[i] = Qs[(4 * ty + i) * LD + x];
#pragma unroll
            for (int j = 0; j < 4; ++j) kv[j] = Ks[(tx + 16 * j) * LD + x];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) sc[i][j] = fmaf(qv[i], kv[j], sc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int row = r0 + 4 * ty + i;
            float mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (j0 + tx + 16 * j > row) sc[i][j] = -INFINITY;  // causal (and keys past L)
                mx = fmaxf(mx, sc[i][j]);
            }
            const float mn = fmaxf(m[i], hmax16(mx));
            const float corr = exp2f(m[i] - mn);  // m = -inf before the first tile -> 0
            float rs = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float p = exp2f(sc[i][j] - mn);
                rs += p;
                Ps[(4 * ty + i) * (kBN + 1) + tx + 16 * j] = p;
            }
            l[i] = l[i] * corr + hsum16(rs);
            m[i] = mn;
#pragma unroll
            for (int c = 0; c < DC; ++c) acc[i][c] *= corr;
        }
        if (!vb) continue;
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kBN; ++kk) {
            float pv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) pv[i] = Ps[(4 * ty + i) * (kBN + 1) + kk];
#pragma unroll
            for (int c = 0; c < DC; ++c) {
                const int x = tx + 16 * c;
                const float vv = x < D ? Vs[kk * D + x] : 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[i][c] = fmaf(pv[i], vv, acc[i][c]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = r0 + 4 * ty + i;
        if (row >= L) continue;
        if (o) {
            T* orow = o + ((size_t)bh * L + row) * D;
            const float inv = 1.f / l[i];
#pragma unroll
            for (int c = 0; c < DC; ++c)
                if (tx + 16 * c < D) st(orow + tx + 16 * c, acc[i][c] * inv);
        }
        if (lse && tx == 0) lse[(size_t)bh * L + row] = (m[i] + log2f(l[i])) * kLn2;
    }
}

// Column sums: a block owns 64 keys of one unit and walks every (query head, query tile I >= J)
// of the unit in a fixed order.  grid (ceil(L/64), units); block 0 = the heaviest key tile.
template <typename T, int D>
__global__ void __launch_bounds__(kST) colsum_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                          const float* __restrict__ lse, float* __restrict__ glo,
                                                          float* __restrict__ loc, int Hq, int Hkv, int G, int L,
                                                          int lwin, float qscale) {
    constexpr int LD = D + 1;
    extern __shared__ float sm[];
    float* Ks = sm;                   // [64 keys][D+1]
    float* Qs = Ks + kBM * LD;        // [64 queries][D+1] scaled
    float* Ls = Qs + kBN * LD;        // [64] lse2 of the query tile
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int J = blockIdx.x, unit = blockIdx.y;
    const int k0 = J * kBM;
    const int b = unit / Hkv, hk = unit % Hkv;
    load_tile<T, D>(Ks, k + (size_t)unit * L * D, k0, L, 1.f);
    const int loc_start = L - lwin;
    const int nqt = (L + kBN - 1) / kBN;
    double ag[4] = {0.0, 0.0, 0.0, 0.0}, al[4] = {0.0, 0.0, 0.0, 0.0};
    for (int h = 0; h < G; ++h) {
        const size_t bh = (size_t)b * Hq + hk * G + h;
        const T* qb = q + bh * L * D;
        for (int I = J; I < nqt; ++I) {
            const int q0 = I * kBN;
            __syncthreads();  // previous tile's Qs / Ls reads done
            load_tile<T, D>(Qs, qb, q0, L, qscale);
            for (int e = tid; e < kBN; e += kST) Ls[e] = q0 + e < L ? lse[bh * L + q0 + e] * kLog2e : 0.f;
            __syncthreads();
            float sc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) sc[i][j] = 0.f;
#pragma unroll 4
            for (int x = 0; x < D; ++x) {
                float kv[4], qv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) kv[i] = Ks[(4 * ty + i) * LD + x];
#pragma unroll
                for (int j = 0; j < 4; ++j) qv[j] = Qs[(tx + 16 * j) * LD + x];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) sc[i][j] = fmaf(kv[i], qv[j], sc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int key = k0 + 4 * ty + i;
                float sg = 0.f, sl = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int qi = q0 + tx + 16 * j;
                    float p = exp2f(sc[i][j] - Ls[tx + 16 * j]);
                    if (qi < key || qi >= L) p = 0.f;
                    sg += p;
                    if (qi >= loc_start) sl += p;
                }
                ag[i] += (double)sg;
                al[i] += (double)sl;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double sg = hsum16(ag[i]), sl = hsum16(al[i]);
        const int key = k0 + 4 * ty + i;
        if (tx == 0 && key < L) {
            glo[(size_t)unit * L + key] = (float)(sg / G);
            loc[(size_t)unit * L + key] = (float)(sl / G);
        }
    }
}

template <typename T, int D>
cudaError_t launch_simt(const Dims& dm, const void* q, const void* k, const void* v, void* o,
                        float* lse, float* glo, float* loc, cudaStream_t s) {
    const float qscale = kLog2e / sqrtf((float)dm.d);
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(fwd_simt_kernel<T, D>), (int)SimtSmem<D>::kFwd);
    if (e == cudaSuccess)
        e = smem_optin(reinterpret_cast<const void*>(colsum_simt_kernel<T, D>), (int)SimtSmem<D>::kCol);
    if (e != cudaSuccess) return e;
    const int nt = (dm.L + kBM - 1) / kBM;
    fwd_simt_kernel<T, D><<<dim3(nt, dm.B * dm.Hq), kST, SimtSmem<D>::kFwd, s>>>(
        (const T*)q, (const T*)k, (const T*)v, (T*)o, lse, dm.Hq, dm.Hkv, dm.G, dm.L, qscale);
    colsum_simt_kernel<T, D><<<dim3(nt, dm.units), kST, SimtSmem<D>::kCol, s>>>(
        (const T*)q, (const T*)k, lse, glo, loc, dm.Hq, dm.Hkv, dm.G, dm.L, dm.lwin_scores, qscale);
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
