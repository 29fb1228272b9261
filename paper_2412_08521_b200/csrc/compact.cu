// compact.cu -- kernel (4): write the fixed-size compressed per-unit cache.
//
// Reference semantics: compress_prefill, proj/src/compressor.cpp:163-242 --
//   keep-all (n <= n_budget, :174-182): every token becomes an exact local;
//   centers (:189-199): slot s = s-th important token in position order, unit key
//     k/|k| (normalized_or_zero :16-25), preserved |k|, raw value, position,
//     score triple (glo, loc_past = loc, loc_cur = 0) (init_score_state,
//     proj/src/scoring.cpp:154-162);
//   locals (:233-235): the last l_win tokens, raw key/value;
//   LUT (:237-240): (position, slot) for important tokens, (position, dest) for
//     merged TBM tokens, (position, -1) for zero-class TBM tokens in zero_class
//     mode (dropped in explicit_removal mode), sorted by position.
// Entries are copied one warp per row with 16-byte vector accesses.
#include "common.cuh"

namespace ems {

namespace {

// Row copy helper: d elements of T, 16-byte vectors when aligned.
template <typename T, int D>
__device__ __forceinline__ void copy_row(T* __restrict__ dst, const T* __restrict__ src, int lane) {
    constexpr int kVec = 16 / sizeof(T);
    if constexpr (D % kVec == 0) {
        const uint4* s = reinterpret_cast<const uint4*>(src);
        uint4* o = reinterpret_cast<uint4*>(dst);
        for (int x = lane; x < D / kVec; x += 32) o[x] = s[x];
    } else {
        for (int x = lane; x < D; x += 32) dst[x] = src[x];
    }
}

template <typename T, int D>
__global__ void __launch_bounds__(256) compact_entries_kernel(
    const T* __restrict__ k, const T* __restrict__ v, int L, const float* __restrict__ glo,
    const float* __restrict__ loc, const int32_t* __restrict__ imp_idx_all,
    const int32_t* __restrict__ counts, int cap_c, int cap_l, int64_t first_pos, T* center_key,
    float* center_norm, T* center_value, int32_t* center_pos, float* center_score, T* local_key,
    T* local_value, int32_t* local_pos, float* local_score) {
    constexpr int R = (D + 31) / 32;
    const int u = blockIdx.y;
    const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int n_imp = counts[4 * u];
    const int n_loc = counts[4 * u + 3];
    const T* kb = k + (size_t)u * L * D;
    const T* vb = v + (size_t)u * L * D;
    if (e < cap_c) {
        if (e >= n_imp) return;
        const int idx = imp_idx_all[(size_t)u * cap_c + e];
        float x[R];
        float ss = 0.f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int dd = lane + 32 * r;
            x[r] = dd < D ? ld(kb + (size_t)idx * D + dd) : 0.f;
            ss = fmaf(x[r], x[r], ss);
        }
        ss = warp_sum(ss);
        const float nrm = sqrtf(ss);
        T* ck = center_key + ((size_t)u * cap_c + e) * D;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int dd = lane + 32 * r;
            if (dd < D) st(ck + dd, nrm > 0.f ? x[r] / nrm : x[r]);
        }
        copy_row<T, D>(center_value + ((size_t)u * cap_c + e) * D, vb + (size_t)idx * D, lane);
        if (lane == 0) {
            center_norm[(size_t)u * cap_c + e] = nrm;
            center_pos[(size_t)u * cap_c + e] = (int32_t)(first_pos + idx);
            float* sc = center_score + ((size_t)u * cap_c + e) * 3;
            sc[0] = glo[(size_t)u * L + idx];
            sc[1] = loc[(size_t)u * L + idx];
            sc[2] = 0.f;
        }
    } else {
        const int l = e - cap_c;
        if (l >= n_loc) return;
        const int idx = L - n_loc + l;
        const size_t o = (size_t)u * cap_l + l;
        copy_row<T, D>(local_key + o * D, kb + (size_t)idx * D, lane);
        copy_row<T, D>(local_value + o * D, vb + (size_t)idx * D, lane);
        if (lane == 0) {
            local_pos[o] = (int32_t)(first_pos + idx);
            float* sc = local_score + o * 3;
            sc[0] = glo[(size_t)u * L + idx];
            sc[1] = loc[(size_t)u * L + idx];
            sc[2] = 0.f;
        }
    }
}

// Position-sorted LUT via a block-wide scan over the class bytes, one CTA per unit.
constexpr int kLutThreads = 1024;
// The kernel ends with HeadCacheState::check_integrity (proj/src/cache.cpp:66-80) on the LUT it
// just wrote: every non-zero-class entry names a live center slot and positions are strictly
// increasing; a violation (possible only through inconsistent caller-supplied stage buffers)
// records EMS_CORRUPTION, the reference's CorruptionError.
__global__ void __launch_bounds__(kLutThreads) compact_lut_kernel(
    int L, const int8_t* __restrict__ cls_all, const int32_t* __restrict__ dest_all,
    const int32_t* __restrict__ counts, int cap_t, int cap_lut, int zero_class, int64_t first_pos,
    int32_t* __restrict__ lut_pos, int32_t* __restrict__ lut_slot, int32_t* __restrict__ out_counts,
    DevStatus* status, int unit_base) {
    __shared__ int shs[32];
    const int u = blockIdx.x, tid = threadIdx.x;
    const int8_t* cls = cls_all + (size_t)u * L;
    const int32_t* dest = dest_all + (size_t)u * cap_t;
    const int per = (L + kLutThreads - 1) / kLutThreads;
    const int s0 = min(L, tid * per), s1 = min(L, s0 + per);
    // pass 1: counts of (important, tbm, lut entries) in this thread's segment.  A TBM
    // token's destination is found through its TBM rank, so ranks are scanned first.
    int ci = 0, ct = 0;
    for (int i = s0; i < s1; ++i) ci += cls[i] == 2, ct += cls[i] == 1;
    const int ri0 = block_incl_scan(ci, shs) - ci;
    const int rt0 = block_incl_scan(ct, shs) - ct;
    int cl = 0;
    {
        int rt = rt0;
        for (int i = s0; i < s1; ++i) {
            if (cls[i] == 2) ++cl;
            else if (cls[i] == 1) cl += (zero_class || (rt < cap_t && dest[rt] >= 0)), ++rt;
        }
    }
    const int cl_incl = block_incl_scan(cl, shs);
    int rl = cl_incl - cl, ri = ri0, rt = rt0;
    int32_t* lp = lut_pos + (size_t)u * cap_lut;
    int32_t* ls = lut_slot + (size_t)u * cap_lut;
    for (int i = s0; i < s1; ++i) {
        if (cls[i] == 2) {
            if (rl < cap_lut) {
                lp[rl] = (int32_t)(first_pos + i);
                ls[rl] = ri;
            }
            ++ri;
            ++rl;
        } else if (cls[i] == 1) {
            const int dd = rt < cap_t ? dest[rt] : -2;
            ++rt;
            if (zero_class || dd >= 0) {
                if (rl < cap_lut) {
                    lp[rl] = (int32_t)(first_pos + i);
                    ls[rl] = dd;  // -1 = zero class; anything < -1 or >= n_centers fails the check
                }
                ++rl;
            }
        }
    }
    const int n_lut = __shfl_sync(0xffffffffu, cl_incl, 31);  // per warp: its last lane's count
    if (tid == kLutThreads - 1) {
        int32_t* oc = out_counts + 4 * u;
        oc[0] = counts[4 * u];
        oc[1] = counts[4 * u + 3];
        oc[2] = cl_incl;  // the last thread's inclusive count = all LUT entries
        oc[3] = 1;
    }
    // check_integrity over the whole LUT (entries written by other threads are visible after
    // the barrier): this thread re-reads its own entries and the one before its first.
    __syncthreads();
    const int n_centers = counts[4 * u];
    const int r0 = cl_incl - cl;
    bool bad = rl > cap_lut;
    for (int r = r0; r < cl_incl && r < cap_lut; ++r) {
        const int sl = ls[r];
        if (sl != -1 && (sl < 0 || sl >= n_centers)) bad = true;  // nonexistent slot
        if (r > 0 && lp[r] <= lp[r - 1]) bad = true;              // not strictly increasing
    }
    (void)n_lut;
    if (bad) record_status(status, EMS_CORRUPTION, unit_base + u);
}

// Keep-all path (n <= n_budget): every token is an exact local; no centers/LUT.
template <typename T, int D>
__global__ void __launch_bounds__(256) keep_all_kernel(const T* __restrict__ k,
                                                       const T* __restrict__ v, int L,
                                                       const float* __restrict__ glo,
                                                       const float* __restrict__ loc, int cap_l,
                                                       int64_t first_pos, T* local_key,
                                                       T* local_value, int32_t* local_pos,
                                                       float* local_score, int32_t* out_counts,
                                                       int32_t* part_counts) {
    const int u = blockIdx.y;
    const int l = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (l == 0 && lane == 0) {
        int32_t* oc = out_counts + 4 * u;
        oc[0] = 0, oc[1] = L, oc[2] = 0, oc[3] = 0;
        if (part_counts) {
            int32_t* pc = part_counts + 4 * u;
            pc[0] = 0, pc[1] = 0, pc[2] = 0, pc[3] = L;
        }
    }
    if (l >= L) return;
    const size_t o = (size_t)u * cap_l + l;
    copy_row<T, D>(local_key + o * D, k + ((size_t)u * L + l) * D, lane);
    copy_row<T, D>(local_value + o * D, v + ((size_t)u * L + l) * D, lane);
    if (lane == 0) {
        local_pos[o] = (int32_t)(first_pos + l);
        float* sc = local_score + o * 3;
        sc[0] = glo[(size_t)u * L + l];
        sc[1] = loc[(size_t)u * L + l];
        sc[2] = 0.f;
    }
}

template <typename T, int D>
cudaError_t launch_compact_t(const Dims& dm, const void* k, const void* v, const float* glo,
                             const float* loc, const ems_stage& sg, const ems_cache& c,
                             int zero_class, int64_t first_pos, DevStatus* status, cudaStream_t s) {
    dim3 ge((dm.cap_c + dm.cap_l + 7) / 8, dm.units);
    compact_entries_kernel<T, D><<<ge, 256, 0, s>>>(
        (const T*)k, (const T*)v, dm.L, glo, loc, sg.imp_idx, sg.part_counts, dm.cap_c, dm.cap_l,
        first_pos, (T*)c.center_key, c.center_norm, (T*)c.center_value, c.center_pos,
        c.center_score, (T*)c.local_key, (T*)c.local_value, c.local_pos, c.local_score);
    compact_lut_kernel<<<dm.units, kLutThreads, 0, s>>>(dm.L, sg.cls, sg.dest, sg.part_counts,
                                                        dm.cap_tbm, dm.cap_lut, zero_class,
                                                        first_pos, c.lut_pos, c.lut_slot, c.counts,
                                                        status, dm.unit_base);
    return cudaGetLastError();
}

template <typename T, int D>
cudaError_t launch_keep_all_t(const Dims& dm, const void* k, const void* v, const float* glo,
                              const float* loc, const ems_stage& sg, const ems_cache& c,
                              int64_t first_pos, cudaStream_t s) {
    dim3 g((dm.L + 7) / 8, dm.units);
    keep_all_kernel<T, D><<<g, 256, 0, s>>>((const T*)k, (const T*)v, dm.L, glo, loc, dm.cap_l,
                                            first_pos, (T*)c.local_key, (T*)c.local_value,
                                            c.local_pos, c.local_score, c.counts, sg.part_counts);
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

cudaError_t launch_compact(const Dims& dm, int dtype, const void* k, const void* v,
                           const float* glo, const float* loc, const ems_stage& sg,
                           const ems_cache& c, int zero_class, int64_t first_pos, DevStatus* status,
                           cudaStream_t s) {
    if (dtype == EMS_F32) {
        EMS_DISPATCH_D(float, launch_compact_t, dm, k, v, glo, loc, sg, c, zero_class, first_pos, status, s)
    } else {
        EMS_DISPATCH_D(__nv_bfloat16, launch_compact_t, dm, k, v, glo, loc, sg, c, zero_class,
                       first_pos, status, s)
    }
}

cudaError_t launch_keep_all(const Dims& dm, int dtype, const void* k, const void* v,
                            const float* glo, const float* loc, const ems_stage& sg,
                            const ems_cache& c, int64_t first_pos, cudaStream_t s) {
    if (dtype == EMS_F32) {
        EMS_DISPATCH_D(float, launch_keep_all_t, dm, k, v, glo, loc, sg, c, first_pos, s)
    } else {
        EMS_DISPATCH_D(__nv_bfloat16, launch_keep_all_t, dm, k, v, glo, loc, sg, c, first_pos, s)
    }
}

}  // namespace ems
