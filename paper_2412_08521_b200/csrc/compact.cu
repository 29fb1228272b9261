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

// Position-sorted LUT as a MERGE of the two ascending index lists select produced (important
// tokens with slots 0..n_imp-1, TBM tokens with their merge destinations), one CTA per unit:
// an entry's LUT index is its rank in its own list plus the number of entries of the other list
// before it (a binary search), so the work is O((n_imp + n_tbm) log) instead of a scan over all
// L class bytes.  In explicit_removal mode the TBM tokens sent to the zero class are dropped: a
// block scan over the TBM list gives the kept prefix.  The kernel ends with
// HeadCacheState::check_integrity (proj/src/cache.cpp:66-80) on the LUT it wrote: every
// non-zero-class entry names a live center slot and positions are strictly increasing; a
// violation (possible only through inconsistent caller-supplied stage buffers) records
// EMS_CORRUPTION, the reference's CorruptionError.
constexpr int kLutThreads = 1024;

__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kLutThreads) compact_lut_kernel(
    const int32_t* __restrict__ imp_idx_all, const int32_t* __restrict__ tbm_idx_all,
    const int32_t* __restrict__ dest_all, const int32_t* __restrict__ counts, int cap_c, int cap_t, int cap_lut,
    int zero_class, int64_t first_pos, int32_t* __restrict__ lut_pos, int32_t* __restrict__ lut_slot,
    int32_t* __restrict__ out_counts, DevStatus* status, int unit_base) {
    __shared__ int shs[32];
    __shared__ int base[kLutThreads];
    __shared__ int s_kept;
    const int u = blockIdx.x, tid = threadIdx.x;
    const int n_imp = counts[4 * u], n_tbm = cap_t > 0 ? counts[4 * u + 1] : 0;
    const int32_t* imp = imp_idx_all + (size_t)u * cap_c;
    const int32_t* tbm = tbm_idx_all + (size_t)u * (cap_t > 0 ? cap_t : 1);
    const int32_t* dest = dest_all + (size_t)u * (cap_t > 0 ? cap_t : 1);
    int32_t* lp = lut_pos + (size_t)u * cap_lut;
    int32_t* ls = lut_slot + (size_t)u * cap_lut;
    auto keep = [&](int b) { return zero_class || dest[b] >= 0; };
    // kept prefix over the TBM list: thread t owns the contiguous chunk [t C, t C + C)
    const int C = (n_tbm + kLutThreads - 1) / kLutThreads;
    const int t0 = min(n_tbm, tid * C), t1 = min(n_tbm, t0 + C);
    int cnt = 0;
    for (int b = t0; b < t1; ++b) cnt += keep(b);
    const int incl = block_incl_scan(cnt, shs);
    base[tid] = incl - cnt;
    if (tid == kLutThreads - 1) s_kept = incl;
    __syncthreads();
    const int n_kept = s_kept, n_lut = n_imp + n_kept;
    auto kept_before = [&](int p) {  // kept TBM entries among tbm[0, p)
        if (p >= n_tbm) return n_kept;
        const int ch = p / C;
        int k = base[ch];
        for (int b = ch * C; b < p; ++b) k += keep(b);
        return k;
    };
    bool bad = n_lut > cap_lut;
    // TBM entries (this thread's chunk, kept ones only)
    for (int b = t0, k = base[tid]; b < t1; ++b) {
        if (!keep(b)) continue;
        const int r = k + lower_bound_i32(imp, n_imp, tbm[b]);
        if (r < cap_lut) {
            lp[r] = (int32_t)(first_pos + tbm[b]);
            ls[r] = dest[b];  // -1 = zero class; anything < -1 or >= n_imp fails the check below
        }
        ++k;
    }
    // important entries: slot a = its rank in position order
    for (int a = tid; a < n_imp; a += kLutThreads) {
        const int r = a + kept_before(lower_bound_i32(tbm, n_tbm, imp[a]));
        if (r < cap_lut) {
            lp[r] = (int32_t)(first_pos + imp[a]);
            ls[r] = a;
        }
    }
    if (tid == 0) {
        int32_t* oc = out_counts + 4 * u;
        oc[0] = n_imp;
        oc[1] = counts[4 * u + 3];
        oc[2] = n_lut;
        oc[3] = 1;
    }
    __syncthreads();
    for (int r = tid; r < n_lut && r < cap_lut; r += kLutThreads) {
        const int sl = ls[r];
        if (sl != -1 && (sl < 0 || sl >= n_imp)) bad = true;  // nonexistent slot
        if (r > 0 && lp[r] <= lp[r - 1]) bad = true;          // not strictly increasing
    }
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
    compact_lut_kernel<<<dm.units, kLutThreads, 0, s>>>(sg.imp_idx, sg.tbm_idx, sg.dest, sg.part_counts, dm.cap_c,
                                                        dm.cap_tbm, dm.cap_lut, zero_class, first_pos, c.lut_pos,
                                                        c.lut_slot, c.counts, status, dm.unit_base);
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
