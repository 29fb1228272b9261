// merge.cu -- kernel (3): redundancy of to-be-merged (TBM) tokens against the
// class centers, argmax destination with zero-class routing; and the
// score-weighted merge of members into their centers (part of kernel (4)).
//
// Reference semantics:
//   redundancy_cross  proj/src/analysis.cpp:51-69 with cos_or_zero :16-24:
//     R[t][c] = clamp(cos(k_t, k_c), -1, 1) * clamp(cos(v_t, v_c), -1, 1) on RAW K/V;
//     a zero-norm token has similarity 0 to everything.  (key_only drops the v factor, D1.)
//   assign_merge_destinations  proj/src/compressor.cpp:76-95: per row the argmax
//     column, strictly-greater wins (ties -> lower column); best >= tau -> column,
//     else kZeroClass (-1).
//   weighted_merge  compressor.cpp:97-161: per center c with members M (ascending
//     TBM order): ws = w_c + sum_M w_i (w = pooled scores, :211, :225);
//     u_c <- normalize((w_c/ws) u_c + sum (w_i/ws) k_i/|k_i|)  (norm and position kept),
//     v_c <- (w_c/ws) v_c + sum (w_i/ws) v_i,  score_c += sum score_i;
//     ws <= 0 -> uniform weights 1/(|M|+1).
#include "common.cuh"

namespace ems {

namespace {

// ---------------------------------------------------------------------------
// Inverse norms of the raw K and V rows of every important and TBM token.
template <typename T, int D>
__global__ void __launch_bounds__(256) norms_kernel(const T* __restrict__ k, const T* __restrict__ v,
                                                    int L, const int32_t* __restrict__ imp_idx,
                                                    const int32_t* __restrict__ tbm_idx,
                                                    const int32_t* __restrict__ counts, int cap_c,
                                                    int cap_t, float* __restrict__ inv_kc,
                                                    float* __restrict__ inv_vc,
                                                    float* __restrict__ inv_kt,
                                                    float* __restrict__ inv_vt) {
    const int u = blockIdx.y;
    const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int n_imp = counts[4 * u], n_tbm = counts[4 * u + 1];
    int idx;
    float *ok, *ov;
    if (e < cap_c) {
        if (e >= n_imp) return;
        idx = imp_idx[(size_t)u * cap_c + e];
        ok = inv_kc + (size_t)u * cap_c + e;
        ov = inv_vc + (size_t)u * cap_c + e;
    } else {
        const int t = e - cap_c;
        if (t >= n_tbm) return;
        idx = tbm_idx[(size_t)u * cap_t + t];
        ok = inv_kt + (size_t)u * cap_t + t;
        ov = inv_vt + (size_t)u * cap_t + t;
    }
    const T* kr = k + ((size_t)u * L + idx) * D;
    const T* vr = v + ((size_t)u * L + idx) * D;
    float sk = 0.f, sv = 0.f;
    for (int x = lane; x < D; x += 32) {
        const float a = ld(kr + x), b = ld(vr + x);
        sk = fmaf(a, a, sk);
        sv = fmaf(b, b, sv);
    }
    sk = warp_sum(sk);
    sv = warp_sum(sv);
    if (lane == 0) {
        *ok = sk > 0.f ? 1.f / sqrtf(sk) : 0.f;
        *ov = sv > 0.f ? 1.f / sqrtf(sv) : 0.f;
    }
}

// ---------------------------------------------------------------------------
// Tiled SIMT similarity + running argmax.  Block: 32 TBM rows x all centers,
// centers staged 32 at a time.  Thread (t = tid/8, g = tid%8) owns centers
// g, g+8, g+16, g+24 of each tile, visited in increasing column order.
template <typename T, int D>
__global__ void __launch_bounds__(256) assign_simt_kernel(
    const T* __restrict__ k, const T* __restrict__ v, int L, const int32_t* __restrict__ imp_idx,
    const int32_t* __restrict__ tbm_idx, const int32_t* __restrict__ counts, int cap_c, int cap_t,
    const float* __restrict__ inv_kc, const float* __restrict__ inv_vc,
    const float* __restrict__ inv_kt, const float* __restrict__ inv_vt, double tau, int key_only,
    int32_t* __restrict__ dest) {
    constexpr int P = D + 1;
    extern __shared__ float sm[];
    float* kt = sm;
    float* vt = kt + 32 * P;
    float* kc = vt + 32 * P;
    float* vc = kc + 32 * P;
    const int u = blockIdx.y;
    const int n_imp = counts[4 * u], n_tbm = counts[4 * u + 1];
    const int t0 = blockIdx.x * 32;
    if (t0 >= n_tbm) return;
    const int tid = threadIdx.x;
    const T* kb = k + (size_t)u * L * D;
    const T* vb = v + (size_t)u * L * D;
    for (int e = tid; e < 32 * D; e += 256) {
        const int r = e / D, x = e % D;
        const int t = t0 + r;
        float a = 0.f, b = 0.f;
        if (t < n_tbm) {
            const int idx = tbm_idx[(size_t)u * cap_t + t];
            a = ld(kb + (size_t)idx * D + x);
            b = ld(vb + (size_t)idx * D + x);
        }
        kt[r * P + x] = a;
        vt[r * P + x] = b;
    }
    const int tr = tid >> 3, g = tid & 7;
    const int t = t0 + tr;
    const float ikt = t < n_tbm ? inv_kt[(size_t)u * cap_t + t] : 0.f;
    const float ivt = t < n_tbm ? inv_vt[(size_t)u * cap_t + t] : 0.f;
    float best = -INFINITY;
    int best_c = 0;
    for (int c0 = 0; c0 < n_imp; c0 += 32) {
        __syncthreads();
        for (int e = tid; e < 32 * D; e += 256) {
            const int r = e / D, x = e % D;
            const int c = c0 + r;
            float a = 0.f, b = 0.f;
            if (c < n_imp) {
                const int idx = imp_idx[(size_t)u * cap_c + c];
                a = ld(kb + (size_t)idx * D + x);
                b = ld(vb + (size_t)idx * D + x);
            }
            kc[r * P + x] = a;
            vc[r * P + x] = b;
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int cl = g + 8 * m;
            const int c = c0 + cl;
            float dk = 0.f, dv = 0.f;
#pragma unroll 8
            for (int x = 0; x < D; ++x) {
                dk = fmaf(kt[tr * P + x], kc[cl * P + x], dk);
                dv = fmaf(vt[tr * P + x], vc[cl * P + x], dv);
            }
            if (c < n_imp) {
                const float ck = fminf(1.f, fmaxf(-1.f, dk * ikt * inv_kc[(size_t)u * cap_c + c]));
                const float cv =
                    key_only ? 1.f : fminf(1.f, fmaxf(-1.f, dv * ivt * inv_vc[(size_t)u * cap_c + c]));
                const float r = ck * cv;
                if (r > best) best = r, best_c = c;  // strict: earliest column wins ties
            }
        }
    }
    // reduce over the 8 threads of the row: larger value, ties -> lower column
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
        if (ob > best || (ob == best && oc < best_c)) best = ob, best_c = oc;
    }
    if (g == 0 && t < n_tbm)
        dest[(size_t)u * cap_t + t] = (n_imp > 0 && (double)best >= tau) ? best_c : -1;
}

// ---------------------------------------------------------------------------
// Weighted merge in two launches.
//
// (a) merge_bucket_kernel, one CTA per unit: the members of every center as a CSR list in
//     ascending TBM order.  Destinations are validated first (anything outside [-1, n_imp)
//     records EMS_CORRUPTION and is treated as the zero class).  The merged tokens' keys
//     (dest << 32 | tbm rank) are collected in shared memory and bitonic-sorted, which gives
//     every bucket its members in ascending TBM order (the reference's accumulation order,
//     compressor.cpp:118-160) without a serial pass; bucket offsets come from an integer
//     histogram and a block scan.  Everything is order-independent integer work, so the
//     output is identical run to run.  Units with more TBM tokens than the sort capacity
//     (kSortCap) fall back to a stable warp-serial fill.
// (b) merge_accum_kernel: one warp per center with members, across (center blocks, units),
//     so the K/V reads of a unit's merges spread over the whole GPU.
constexpr int kBucketThreads = 1024;
constexpr int kSortCap = 16384;  // keys per unit sorted in shared memory (128 KB)

__global__ void __launch_bounds__(kBucketThreads) merge_bucket_kernel(
    const int32_t* __restrict__ counts, const int32_t* __restrict__ dest_all, int cap_c, int cap_t,
    int32_t* __restrict__ ws_off, int32_t* __restrict__ ws_members, DevStatus* status, int unit_base) {
    extern __shared__ unsigned long long keys[];  // [sort capacity]
    __shared__ int sh[32];
    __shared__ int n_merged, bad;
    const int u = blockIdx.x, tid = threadIdx.x;
    const int n_imp = counts[4 * u], n_tbm = counts[4 * u + 1];
    const int32_t* dest = dest_all + (size_t)u * cap_t;
    int32_t* off = ws_off + (size_t)u * (cap_c + 1);
    int32_t* mem = ws_members + (size_t)u * cap_t;
    if (tid == 0) n_merged = 0, bad = 0;
    for (int c = tid; c <= n_imp; c += kBucketThreads) off[c] = 0;
    __syncthreads();
    // histogram of destinations (integer atomics: order-independent) + collection of the keys
    const bool sortable = n_tbm <= kSortCap;
    for (int t = tid; t < n_tbm; t += kBucketThreads) {
        const int d = dest[t];
        if (d < -1 || d >= n_imp) {
            bad = 1;
            continue;
        }
        if (d < 0) continue;
        atomicAdd(&off[d + 1], 1);
        if (sortable) keys[atomicAdd(&n_merged, 1)] = ((unsigned long long)d << 32) | (unsigned)t;
    }
    __syncthreads();
    if (bad && tid == 0) record_status(status, EMS_CORRUPTION, unit_base + u);
    // exclusive bucket offsets: off[c] = start of bucket c, off[n_imp] = all merged tokens
    {
        const int per = (n_imp + kBucketThreads) / kBucketThreads;  // n_imp + 1 entries
        const int c0 = min(n_imp + 1, tid * per), c1 = min(n_imp + 1, c0 + per);
        int run = 0;
        for (int c = c0; c < c1; ++c) run += off[c];
        int base = block_incl_scan(run, sh) - run;
        for (int c = c0; c < c1; ++c) {
            base += off[c];
            off[c] = base;  // inclusive over [0, c] of the shifted counts = start of bucket c
        }
    }
    __syncthreads();
    if (sortable) {
        const int m = n_merged;
        int n = 1;
        while (n < m) n <<= 1;
        for (int i = m + tid; i < n; i += kBucketThreads) keys[i] = ~0ull;
        __syncthreads();
        for (int k = 2; k <= n; k <<= 1)  // bitonic sort, ascending (dest, t)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < n; i += kBucketThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long a = keys[i], b = keys[ixj];
                        const bool up = (i & k) == 0;
                        if ((a > b) == up) {
                            keys[i] = b;
                            keys[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        for (int i = tid; i < m; i += kBucketThreads) mem[i] = (int32_t)(keys[i] & 0xffffffffull);
    } else if (tid < 32) {  // stable warp-serial fill with per-bucket cursors
        const int lane = tid;
        int32_t* cur = off;  // the bucket starts double as cursors
        for (int base = 0; base < n_tbm; base += 32) {
            const int t = base + lane;
            int dd = t < n_tbm ? dest[t] : -1;
            if (dd >= n_imp || dd < -1) dd = -1;
            const unsigned act = __ballot_sync(0xffffffffu, dd >= 0);
            if (dd >= 0) {
                const unsigned same = __match_any_sync(act, dd);
                const int rank = __popc(same & ((1u << lane) - 1u));
                const int pos = cur[dd];
                mem[pos + rank] = t;
                __syncwarp(act);
                if (rank == 0) cur[dd] = pos + __popc(same);
            }
            __syncwarp();
        }
    }
    if (!sortable) {  // the cursors now hold bucket ends (end of c == start of c + 1): shift back
        __syncthreads();
        if (tid == 0) {
            for (int c = n_imp; c > 0; --c) off[c] = off[c - 1];
            off[0] = 0;
        }
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) merge_accum_kernel(
    const T* __restrict__ k, const T* __restrict__ v, int L, const float* __restrict__ glo,
    const float* __restrict__ loc, const float* __restrict__ pooled_all,
    const int32_t* __restrict__ imp_idx_all, const int32_t* __restrict__ tbm_idx_all,
    const int32_t* __restrict__ counts, int cap_c, int cap_t, const int32_t* __restrict__ ws_off,
    const int32_t* __restrict__ ws_members, T* __restrict__ center_key, T* __restrict__ center_value,
    float* __restrict__ center_score) {
    constexpr int R = (D + 31) / 32;
    const int u = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int n_imp = counts[4 * u];
    if (c >= n_imp || counts[4 * u + 1] == 0) return;
    const int32_t* off = ws_off + (size_t)u * (cap_c + 1);
    const int b0 = off[c], b1 = off[c + 1];
    if (b1 == b0) return;
    const int32_t* mem = ws_members + (size_t)u * cap_t;
    const int32_t* tbm_idx = tbm_idx_all + (size_t)u * cap_t;
    const float* pooled = pooled_all + (size_t)u * L;
    const T* kb = k + (size_t)u * L * D;
    const T* vb = v + (size_t)u * L * D;
    const int ci = imp_idx_all[(size_t)u * cap_c + c];
    double ws = (double)pooled[ci];
    for (int m = b0; m < b1; ++m) ws += (double)pooled[tbm_idx[mem[m]]];
    const double uniform = 1.0 / (double)(b1 - b0 + 1);
    float mk[R], mv[R], x[R];
    // the center's own unit key and value first, then the members in ascending TBM order
    float ss = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int dd = lane + 32 * r;
        x[r] = dd < D ? ld(kb + (size_t)ci * D + dd) : 0.f;
        ss = fmaf(x[r], x[r], ss);
    }
    ss = warp_sum(ss);
    float nrm = sqrtf(ss);
    float w = (float)(ws > 0.0 ? (double)pooled[ci] / ws : uniform);
    float sg = glo[(size_t)u * L + ci], sl = loc[(size_t)u * L + ci];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int dd = lane + 32 * r;
        const float uk = nrm > 0.f ? x[r] / nrm : x[r];
        mk[r] = w * uk;
        mv[r] = dd < D ? w * ld(vb + (size_t)ci * D + dd) : 0.f;
    }
    for (int m = b0; m < b1; ++m) {
        const int ti = tbm_idx[mem[m]];
        ss = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int dd = lane + 32 * r;
            x[r] = dd < D ? ld(kb + (size_t)ti * D + dd) : 0.f;
            ss = fmaf(x[r], x[r], ss);
        }
        ss = warp_sum(ss);
        nrm = sqrtf(ss);
        w = (float)(ws > 0.0 ? (double)pooled[ti] / ws : uniform);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int dd = lane + 32 * r;
            const float uk = nrm > 0.f ? x[r] / nrm : x[r];
            mk[r] = fmaf(w, uk, mk[r]);
            if (dd < D) mv[r] = fmaf(w, ld(vb + (size_t)ti * D + dd), mv[r]);
        }
        sg += glo[(size_t)u * L + ti];
        sl += loc[(size_t)u * L + ti];
    }
    ss = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) ss = fmaf(mk[r], mk[r], ss);
    ss = warp_sum(ss);
    const float mn = sqrtf(ss);
    T* ck = center_key + ((size_t)u * cap_c + c) * D;
    T* cv = center_value + ((size_t)u * cap_c + c) * D;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int dd = lane + 32 * r;
        if (dd < D) {
            // mn == 0 keeps the center's current unit key (compressor.cpp:152-158)
            if (mn > 0.f) st(ck + dd, mk[r] / mn);
            st(cv + dd, mv[r]);
        }
    }
    if (lane == 0) {
        float* sc = center_score + ((size_t)u * cap_c + c) * 3;
        sc[0] = sg;
        sc[1] = sl;
        sc[2] = 0.f;
    }
}

template <typename T, int D>
cudaError_t launch_merge_assign_t(const Dims& dm, const void* k, const void* v,
                                  const ems_stage& sg, double tau, int key_only, float* inv_kc,
                                  float* inv_vc, float* inv_kt, float* inv_vt, cudaStream_t s) {
    dim3 gn((dm.cap_c + dm.cap_tbm + 7) / 8, dm.units);
    norms_kernel<T, D><<<gn, 256, 0, s>>>((const T*)k, (const T*)v, dm.L, sg.imp_idx, sg.tbm_idx,
                                         sg.part_counts, dm.cap_c, dm.cap_tbm, inv_kc, inv_vc,
                                         inv_kt, inv_vt);
    const size_t smem = sizeof(float) * 4 * 32 * (D + 1);
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(assign_simt_kernel<T, D>), (int)smem);
    if (e != cudaSuccess) return e;
    dim3 ga((dm.cap_tbm + 31) / 32, dm.units);
    if (dm.cap_tbm > 0)
        assign_simt_kernel<T, D><<<ga, 256, smem, s>>>(
            (const T*)k, (const T*)v, dm.L, sg.imp_idx, sg.tbm_idx, sg.part_counts, dm.cap_c,
            dm.cap_tbm, inv_kc, inv_vc, inv_kt, inv_vt, tau, key_only, sg.dest);
    return cudaGetLastError();
}

template <typename T, int D>
cudaError_t launch_merge_scatter_t(const Dims& dm, const void* k, const void* v, const float* glo,
                                   const float* loc, const ems_stage& sg, int32_t* ws_off,
                                   int32_t* ws_members, const ems_cache& cache, DevStatus* status,
                                   cudaStream_t s) {
    int n = 1;
    while (n < dm.cap_tbm && n < kSortCap) n <<= 1;
    const int smem = (int)(sizeof(unsigned long long) * n);
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(merge_bucket_kernel), smem);
    if (e != cudaSuccess) return e;
    merge_bucket_kernel<<<dm.units, kBucketThreads, smem, s>>>(sg.part_counts, sg.dest, dm.cap_c, dm.cap_tbm,
                                                               ws_off, ws_members, status, dm.unit_base);
    merge_accum_kernel<T, D><<<dim3((dm.cap_c + 7) / 8, dm.units), 256, 0, s>>>(
        (const T*)k, (const T*)v, dm.L, glo, loc, sg.pooled, sg.imp_idx, sg.tbm_idx, sg.part_counts, dm.cap_c,
        dm.cap_tbm, ws_off, ws_members, (T*)cache.center_key, (T*)cache.center_value, cache.center_score);
    return cudaGetLastError();
}

}  // namespace

#define EMS_DISPATCH_D(T, FN, ...)                              \
    switch (dm.d) {                                             \
        case 8: return FN<T, 8>(__VA_ARGS__);                   \
        case 16: return FN<T, 16>(__VA_ARGS__);                 \
        case 32: return FN<T, 32>(__VA_ARGS__);                 \
        case 64: return FN<T, 64>(__VA_ARGS__);                 \
        case 96: return FN<T, 96>(__VA_ARGS__);                 \
        case 128: return FN<T, 128>(__VA_ARGS__);               \
        default: return cudaErrorInvalidValue;                  \
    }

cudaError_t launch_merge_assign(const Dims& dm, int dtype, const void* k, const void* v,
                                const ems_stage& sg, double tau, int key_only, float* inv_kc,
                                float* inv_vc, float* inv_kt, float* inv_vt, cudaStream_t s) {
    if (dtype == EMS_F32) {
        EMS_DISPATCH_D(float, launch_merge_assign_t, dm, k, v, sg, tau, key_only, inv_kc, inv_vc,
                       inv_kt, inv_vt, s)
    } else {
        EMS_DISPATCH_D(__nv_bfloat16, launch_merge_assign_t, dm, k, v, sg, tau, key_only, inv_kc,
                       inv_vc, inv_kt, inv_vt, s)
    }
}

cudaError_t launch_merge_scatter(const Dims& dm, int dtype, const void* k, const void* v,
                                 const float* glo, const float* loc, const ems_stage& sg,
                                 int32_t* ws_count, int32_t* ws_members, const ems_cache& cache,
                                 DevStatus* status, cudaStream_t s) {
    if (dtype == EMS_F32) {
        EMS_DISPATCH_D(float, launch_merge_scatter_t, dm, k, v, glo, loc, sg, ws_count, ws_members,
                       cache, status, s)
    } else {
        EMS_DISPATCH_D(__nv_bfloat16, launch_merge_scatter_t, dm, k, v, glo, loc, sg, ws_count,
                       ws_members, cache, status, s)
    }
}

}  // namespace ems

namespace ems {
namespace {
// Standalone redundancy_cross (analysis.cpp:51-69): one warp per row, all columns.
template <typename T>
__global__ void __launch_bounds__(256) redundancy_cross_kernel(const T* kr, const T* vr, int nr,
                                                               const T* kc, const T* vc, int nc,
                                                               int d, int key_only, float* out) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= nr) return;
    float sk = 0.f, sv = 0.f;
    for (int x = lane; x < d; x += 32) {
        const float a = ld(kr + (size_t)row * d + x), b = ld(vr + (size_t)row * d + x);
        sk = fmaf(a, a, sk), sv = fmaf(b, b, sv);
    }
    const float nk = sqrtf(warp_sum(sk)), nv = sqrtf(warp_sum(sv));
    for (int c = 0; c < nc; ++c) {
        float dk = 0.f, dv = 0.f, ck2 = 0.f, cv2 = 0.f;
        for (int x = lane; x < d; x += 32) {
            const float a = ld(kr + (size_t)row * d + x), b = ld(vr + (size_t)row * d + x);
            const float e = ld(kc + (size_t)c * d + x), f = ld(vc + (size_t)c * d + x);
            dk = fmaf(a, e, dk), dv = fmaf(b, f, dv), ck2 = fmaf(e, e, ck2), cv2 = fmaf(f, f, cv2);
        }
        dk = warp_sum(dk), dv = warp_sum(dv);
        const float nck = sqrtf(warp_sum(ck2)), ncv = sqrtf(warp_sum(cv2));
        const float cosk = (nk == 0.f || nck == 0.f) ? 0.f : fminf(1.f, fmaxf(-1.f, dk / (nk * nck)));
        const float cosv = (nv == 0.f || ncv == 0.f) ? 0.f : fminf(1.f, fmaxf(-1.f, dv / (nv * ncv)));
        if (lane == 0) out[(size_t)row * nc + c] = key_only ? cosk : cosk * cosv;
    }
}
}  // namespace

cudaError_t launch_redundancy_cross(int dtype, int d, const void* kr, const void* vr, int nr,
                                    const void* kc, const void* vc, int nc, int key_only,
                                    float* r, cudaStream_t s) {
    const int grid = (nr + 7) / 8;
    if (dtype == EMS_F32)
        redundancy_cross_kernel<float><<<grid, 256, 0, s>>>((const float*)kr, (const float*)vr, nr,
                                                            (const float*)kc, (const float*)vc, nc,
                                                            d, key_only, r);
    else
        redundancy_cross_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
            (const __nv_bfloat16*)kr, (const __nv_bfloat16*)vr, nr, (const __nv_bfloat16*)kc,
            (const __nv_bfloat16*)vc, nc, d, key_only, r);
    return cudaGetLastError();
}
}  // namespace ems
