// select.cu -- kernel (2): scale alignment + combine + mean-pool + exact top-k
// partition of the candidate tokens, one CTA per unit.  The baseline policies
// (policies.cpp:141-176) replace the ranked score: glo (H2O), mean-pooled loc (SnapKV),
// or a sinks + recent-window indicator (StreamingLLM); they have no TBM set.
//
// Reference semantics (all per head/unit):
//   effective_score  proj/src/scoring.cpp:146-152 ->
//     combine_glo_loc  scoring.cpp:105-124: align = sum(loc)/sum(glo) over ALL L tokens,
//                      s_i = max(glo_i * align, loc_i);  sum(glo) <= 0 -> DegenerateInputError
//     mean_pool_1d     numerics.cpp:62-82: centred window, truncated at the edges
//   clamp_kernel       compressor.cpp:29-34 (done on the host)
//   partition_tokens   compressor.cpp:48-74: candidates [0, L-w); stable sort by
//                      pooled desc (ties -> lower index); top n_imp important, next
//                      n_tbm to-be-merged, rest irrelevant; each set ascending.
//
// The stable-sort order is reproduced exactly by ranking the unique 64-bit key
//   key_i = (bits(pooled_i as f32) << 32) | (0xFFFFFFFF - i)
// (pooled >= 0, so f32 bit patterns order like the values; the low word breaks
// ties toward the lower index).  An MSD radix select (8 passes of 8 bits, two
// targets at once) finds the n_imp-th and (n_imp+n_tbm)-th largest keys; every
// token is then classified by comparison, and ascending index lists come out of
// a block-wide prefix sum.  Integer histograms make the result deterministic.
#include <stdlib.h>

#include "common.cuh"

namespace ems {

namespace {

constexpr int kSelThreads = 1024;

// A unit whose scores have no global mass (the reference throws DegenerateInputError,
// scoring.cpp:115-117) still leaves a valid stage behind, so the merge / compact kernels that
// follow in the same pipeline only see consistent data (no centers, no TBM tokens, no LUT; the
// exact locals): every candidate irrelevant, counts {0, 0, n_cand, l_win}.  The error itself is
// reported through the device status word (ems_sync_status).
__device__ void write_empty_partition(int8_t* cls, int32_t* counts, int L, int l_win, int i0, int i1, int tid,
                                      int nthreads) {
    const int n_cand = L - l_win;
    for (int i = i0 + tid; i < i1; i += nthreads) cls[i] = i < n_cand ? 0 : 3;
    if (counts && tid == 0) {
        counts[0] = 0;
        counts[1] = 0;
        counts[2] = n_cand;
        counts[3] = l_win;
    }
}
constexpr int kSelWarps = kSelThreads / 32;

__device__ __forceinline__ unsigned long long sel_key(const float* pooled, int i) {
    return ((unsigned long long)__float_as_uint(pooled[i]) << 32) |
           (unsigned long long)(0xFFFFFFFFu - (unsigned)i);
}

// Block-wide fixed-order sum of per-thread doubles (deterministic).
__device__ double block_sum(double v, double* sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum(v);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < kSelWarps ? sh[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) sh[0] = t;
    }
    __syncthreads();
    t = sh[0];
    __syncthreads();
    return t;
}

// Given a 256-bin histogram and a 1-based rank `rem` counted from the top bin,
// returns the bin holding that rank and the count strictly above it (one warp).
__device__ void find_bin(const int* hist, int rem, int* out_bin, int* out_above) {
    const int lane = threadIdx.x & 31;
    // lane l owns bins 255-8l ... 248-8l (descending)
    int c[8], tot = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = hist[255 - 8 * lane - t], tot += c[t];
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    const int excl = incl - tot;
    const unsigned ballot = __ballot_sync(0xffffffffu, excl < rem && rem <= incl);
    const int owner = __ffs(ballot) - 1;
    if (lane == owner) {
        int run = excl;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (run < rem && rem <= run + c[t]) {
                *out_bin = 255 - 8 * lane - t;
                *out_above = run;
                break;
            }
            run += c[t];
        }
    }
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(
    const float* __restrict__ glo, const float* __restrict__ loc, int L, int l_win, int n_imp,
    int n_tbm, int kernel, float* __restrict__ pooled_all, int8_t* __restrict__ cls_all,
    int32_t* __restrict__ imp_idx_all, int32_t* __restrict__ tbm_idx_all,
    int32_t* __restrict__ counts_all, int cap_c, int cap_tbm, DevStatus* status, int unit_base,
    int policy, int sink, int n_budget) {
    __shared__ double sh[32];
    __shared__ int hist[2][256];
    __shared__ int sel_bin[2], sel_above[2], sel_one[2];
    __shared__ unsigned long long hkey[2][256];
    __shared__ int scan[2][kSelThreads];
    __shared__ int degenerate;
    const int u = blockIdx.x;
    const int tid = threadIdx.x;
    const float* g = glo + (size_t)u * L;
    const float* lo = loc + (size_t)u * L;
    float* pooled = pooled_all + (size_t)u * L;

    const int half = kernel / 2;
    if (policy != EMS_POLICY_EMS) {
        // baseline policies (policies.cpp:141-176): the ranked score, no combine / alignment
        const int n_cand_b = L - l_win;
        const int lo_recent = max(L - (n_budget - sink), sink);
        for (int i = tid; i < L; i += kSelThreads) {
            float v;
            if ((policy == EMS_POLICY_H2O || policy == kPolicyPooled)) {
                v = g[i];  // top_k_by(scores.glo, ...)
            } else if (policy == EMS_POLICY_SNAPKV) {  // mean_pool_1d(loc_past + loc_cur)
                const int a = max(0, i - half), bnd = min(L - 1, i + half);
                double acc = 0.0;
                for (int jj = a; jj <= bnd; ++jj) acc += (double)lo[jj];
                v = (float)(acc / (double)(bnd - a + 1));
            } else {  // streaming_llm: sinks + the recent window, as an indicator score
                v = (i < sink || (i >= lo_recent && i < n_cand_b)) ? 1.f : 0.f;
            }
            pooled[i] = v;
        }
        __syncthreads();
    } else {
    // 1. alignment sums over all L tokens (fp64)
    double sg = 0.0, sl = 0.0;
    for (int i = tid; i < L; i += kSelThreads) sg += (double)g[i], sl += (double)lo[i];
    sg = block_sum(sg, sh);
    sl = block_sum(sl, sh);
    if (tid == 0) degenerate = !(sg > 0.0);
    __syncthreads();
    if (degenerate) {  // DegenerateInputError (scoring.cpp:115-117); leave a valid empty partition
        if (tid == 0) record_status(status, EMS_DEGENERATE_INPUT, unit_base + u);
        write_empty_partition(cls_all + (size_t)u * L, counts_all + 4 * u, L, l_win, 0, L, tid, kSelThreads);
        return;
    }
    const double align = sl / sg;

    // 2. combine + centred mean pool with truncated edges (fp64), stored as f32
    for (int i = tid; i < L; i += kSelThreads) {
        const int a = max(0, i - half), bnd = min(L - 1, i + half);
        double acc = 0.0;
        for (int jj = a; jj <= bnd; ++jj) {
            const double x = (double)g[jj] * align, y = (double)lo[jj];
            acc += x > y ? x : y;
        }
        pooled[i] = (float)(acc / (double)(bnd - a + 1));
    }
    __syncthreads();
    }

    // 3. radix select of the k1-th and k2-th largest candidate keys
    const int n_cand = L - l_win;
    const int k1 = n_imp, k2 = n_imp + n_tbm;
    // MSD radix select over the 64-bit keys, both cuts at once.  A bin that holds exactly one
    // key resolves its cut: that key (recorded next to the histogram) is the cut, and the
    // remaining passes are skipped (random fp32 scores typically resolve after 3 of the 8).
    unsigned long long pre[2] = {0ull, 0ull};
    int rem[2] = {k1, k2};
    bool res[2] = {false, false};
    for (int pass = 0; pass < 8 && !(res[0] && res[1]); ++pass) {
        const int shift = 56 - 8 * pass;
        const unsigned long long hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (int e = tid; e < 512; e += kSelThreads) (&hist[0][0])[e] = 0;
        __syncthreads();
        for (int i = tid; i < n_cand; i += kSelThreads) {
            const unsigned long long key = sel_key(pooled, i);
            const int bin = (int)((key >> shift) & 255ull);
#pragma unroll
            for (int t = 0; t < 2; ++t)
                if (!res[t] && (key & hi_mask) == pre[t]) {
                    atomicAdd(&hist[t][bin], 1);
                    hkey[t][bin] = key;  // racy unless the bin ends up holding one key
                }
        }
        __syncthreads();
        const int warp = tid >> 5;
        if (warp < 2 && !res[warp]) {
            find_bin(hist[warp], rem[warp], &sel_bin[warp], &sel_above[warp]);
            __syncwarp();
            if ((tid & 31) == 0) sel_one[warp] = hist[warp][sel_bin[warp]] == 1;
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (res[t]) continue;
            pre[t] |= (unsigned long long)sel_bin[t] << shift;
            rem[t] -= sel_above[t];
            if (sel_one[t]) {
                pre[t] = hkey[t][sel_bin[t]];
                res[t] = true;
            }
        }
        __syncthreads();
    }
    const unsigned long long T1 = pre[0];
    const unsigned long long T2 = n_tbm > 0 ? pre[1] : pre[0];

    // 4. classify + ascending index lists via a block-wide exclusive scan
    int8_t* cls = cls_all + (size_t)u * L;
    int32_t* imp_idx = imp_idx_all + (size_t)u * cap_c;
    int32_t* tbm_idx = tbm_idx_all + (size_t)u * cap_tbm;
    const int per = (L + kSelThreads - 1) / kSelThreads;
    const int s0 = min(L, tid * per), s1 = min(L, s0 + per);
    int ci = 0, ct = 0;
    for (int i = s0; i < s1; ++i) {
        if (i < n_cand) {
            const unsigned long long key = sel_key(pooled, i);
            ci += key >= T1;
            ct += (key < T1 && key >= T2);
        }
    }
    scan[0][tid] = ci;
    scan[1][tid] = ct;
    __syncthreads();
    // Hillis-Steele inclusive scan (1024 entries, two arrays)
    for (int o = 1; o < kSelThreads; o <<= 1) {
        const int a = tid >= o ? scan[0][tid - o] : 0;
        const int b = tid >= o ? scan[1][tid - o] : 0;
        __syncthreads();
        scan[0][tid] += a;
        scan[1][tid] += b;
        __syncthreads();
    }
    int ri = scan[0][tid] - ci, rt = scan[1][tid] - ct;
    for (int i = s0; i < s1; ++i) {
        int8_t c = 3;
        if (i < n_cand) {
            const unsigned long long key = sel_key(pooled, i);
            if (key >= T1) {
                c = 2;
                imp_idx[ri++] = i;
            } else if (key >= T2) {
                c = 1;
                tbm_idx[rt++] = i;
            } else {
                c = 0;
            }
        }
        cls[i] = c;
    }
    if (tid == 0) {
        int32_t* cnt = counts_all + 4 * u;
        cnt[0] = n_imp;
        cnt[1] = n_tbm;
        cnt[2] = n_cand - n_imp - n_tbm;
        cnt[3] = l_win;
    }
}

// ---------------------------------------------------------------------------------------
// Cluster version: kClu CTAs per unit, each owning a contiguous slice of the tokens.  The
// fp64 alignment sums, the radix histograms and the index-list offsets are exchanged through
// distributed shared memory and always combined in rank order, so the result is identical to
// the single-CTA kernel (same keys, same cut values, same ascending lists).
constexpr int kClu = 8;
constexpr int kCThreads = 512;

__device__ double cblock_sum(double v, double* sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < kCThreads / 32; ++i) t += sh[i];
    __syncthreads();
    return t;
}

__global__ void __cluster_dims__(kClu, 1, 1) __launch_bounds__(kCThreads) select_cluster_kernel(
    const float* __restrict__ glo, const float* __restrict__ loc, int L, int l_win, int n_imp, int n_tbm,
    int kernel, float* __restrict__ pooled_all, int8_t* __restrict__ cls_all, int32_t* __restrict__ imp_idx_all,
    int32_t* __restrict__ tbm_idx_all, int32_t* __restrict__ counts_all, int cap_c, int cap_tbm, DevStatus* status,
    int unit_base, int policy, int sink, int n_budget) {
    __shared__ double sh[32];
    __shared__ double s_part[2];           // this CTA's alignment partials (read remotely)
    __shared__ int hist[2][2][256];        // [parity][target][bin] (read remotely)
    __shared__ long long hkey[2][2][256];  // [parity][target][bin]: a key of that bin (read remotely)
    __shared__ long long sel_key_v[2];
    __shared__ int sel_one[2];
    __shared__ int s_cnt[2];               // this CTA's important / TBM counts (read remotely)
    __shared__ int scan[2][kCThreads];
    __shared__ int sel_bin[2], sel_above[2];
    const int rank = (int)cl_rank();
    const int u = blockIdx.x / kClu;
    const int tid = threadIdx.x;
    const float* g = glo + (size_t)u * L;
    const float* lo = loc + (size_t)u * L;
    float* pooled = pooled_all + (size_t)u * L;
    const int per_cta = (L + kClu - 1) / kClu;
    const int c0 = min(L, rank * per_cta), c1 = min(L, c0 + per_cta);
    const int half = kernel / 2;
    // 1. pooled score of this CTA's slice (+ 2. alignment over all L tokens for EMS)
    double align = 0.0;
    if (policy == EMS_POLICY_EMS) {
        double sg = 0.0, sl = 0.0;
        for (int i = c0 + tid; i < c1; i += kCThreads) sg += (double)g[i], sl += (double)lo[i];
        sg = cblock_sum(sg, sh);
        sl = cblock_sum(sl, sh);
        if (tid == 0) s_part[0] = sg, s_part[1] = sl;
        cl_sync();
        double tg = 0.0, tl = 0.0;
        for (int r = 0; r < kClu; ++r) tg += ld_dsm_f64(&s_part[0], r), tl += ld_dsm_f64(&s_part[1], r);
        if (!(tg > 0.0)) {  // DegenerateInputError; leave a valid empty partition
            if (tid == 0 && rank == 0) record_status(status, EMS_DEGENERATE_INPUT, unit_base + u);
            write_empty_partition(cls_all + (size_t)u * L, rank == 0 ? counts_all + 4 * u : nullptr, L, l_win, c0,
                                  c1, tid, kCThreads);
            cl_sync();
            return;
        }
        align = tl / tg;
    }
    const int n_cand_b = L - l_win;
    const int lo_recent = max(L - (n_budget - sink), sink);
    for (int i = c0 + tid; i < c1; i += kCThreads) {
        float v;
        if ((policy == EMS_POLICY_H2O || policy == kPolicyPooled)) {
            v = g[i];
        } else if (policy == EMS_POLICY_STREAMING) {
            v = (i < sink || (i >= lo_recent && i < n_cand_b)) ? 1.f : 0.f;
        } else {
            const int a = max(0, i - half), bnd = min(L - 1, i + half);
            double acc = 0.0;
            for (int jj = a; jj <= bnd; ++jj) {
                if (policy == EMS_POLICY_SNAPKV) {
                    acc += (double)lo[jj];
                } else {
                    const double x = (double)g[jj] * align, y = (double)lo[jj];
                    acc += x > y ? x : y;
                }
            }
            v = (float)(acc / (double)(bnd - a + 1));
        }
        pooled[i] = v;
    }
    __syncthreads();
    // 3. radix select of the k1-th / k2-th largest candidate keys, histograms summed over the cluster
    const int n_cand = L - l_win;
    const int e0 = min(n_cand, c0), e1 = min(n_cand, c1);
    unsigned long long pre[2] = {0ull, 0ull};
    int rem[2] = {n_imp, n_imp + n_tbm};
    bool res[2] = {false, false};  // cut resolved early (a bin holding exactly one key)
    for (int pass = 0; pass < 8 && !(res[0] && res[1]); ++pass) {
        const int par = pass & 1;
        const int shift = 56 - 8 * pass;
        const unsigned long long hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (int e = tid; e < 512; e += kCThreads) (&hist[par][0][0])[e] = 0;
        __syncthreads();
        for (int i = e0 + tid; i < e1; i += kCThreads) {
            const unsigned long long key = sel_key(pooled, i);
            const int bin = (int)((key >> shift) & 255ull);
#pragma unroll
            for (int t = 0; t < 2; ++t)
                if (!res[t] && (key & hi_mask) == pre[t]) {
                    atomicAdd(&hist[par][t][bin], 1);
                    hkey[par][t][bin] = (long long)key;  // racy unless this CTA holds one key there
                }
        }
        cl_sync();  // every CTA's histogram complete (and last pass's reads done: other parity)
        // global histogram = sum over the cluster, in rank order (all CTAs compute the same)
        for (int e = tid; e < 512; e += kCThreads) {
            int tsum = 0;
            for (int r = 0; r < kClu; ++r) tsum += ld_dsm_i32(&hist[par][0][0] + e, r);
            scan[0][e] = tsum;  // scan[0] reused as a 512-entry staging area
        }
        __syncthreads();
        const int warp = tid >> 5;
        if (warp < 2 && !res[warp]) {
            find_bin(&scan[0][256 * warp], rem[warp], &sel_bin[warp], &sel_above[warp]);
            __syncwarp();
            if ((tid & 31) == 0) {
                const int bin = sel_bin[warp];
                sel_one[warp] = scan[0][256 * warp + bin] == 1;
                if (sel_one[warp])  // the single key lives in the one CTA whose count is 1
                    for (int r = 0; r < kClu; ++r)
                        if (ld_dsm_i32(&hist[par][warp][bin], r) == 1) sel_key_v[warp] = ld_dsm_i64(&hkey[par][warp][bin], r);
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (res[t]) continue;
            pre[t] |= (unsigned long long)sel_bin[t] << shift;
            rem[t] -= sel_above[t];
            if (sel_one[t]) {
                pre[t] = (unsigned long long)sel_key_v[t];
                res[t] = true;
            }
        }
        __syncthreads();
    }
    const unsigned long long T1 = pre[0];
    const unsigned long long T2 = n_tbm > 0 ? pre[1] : pre[0];
    // 4. classify; ascending lists: CTA offset = counts of lower ranks, then a block scan
    const int per = (c1 - c0 + kCThreads - 1) / kCThreads;
    const int s0 = min(c1, c0 + tid * per), s1 = min(c1, s0 + per);
    int ci = 0, ct = 0;
    for (int i = s0; i < s1; ++i)
        if (i < n_cand) {
            const unsigned long long key = sel_key(pooled, i);
            ci += key >= T1;
            ct += (key < T1 && key >= T2);
        }
    __shared__ int shs[32];
    const int inc_i = block_incl_scan(ci, shs);
    const int inc_t = block_incl_scan(ct, shs);
    if (tid == kCThreads - 1) s_cnt[0] = inc_i, s_cnt[1] = inc_t;
    cl_sync();
    int bi = 0, bt = 0;
    for (int r = 0; r < rank; ++r) bi += ld_dsm_i32(&s_cnt[0], r), bt += ld_dsm_i32(&s_cnt[1], r);
    int8_t* cls = cls_all + (size_t)u * L;
    int32_t* imp_idx = imp_idx_all + (size_t)u * cap_c;
    int32_t* tbm_idx = tbm_idx_all + (size_t)u * cap_tbm;
    int ri = bi + inc_i - ci, rt = bt + inc_t - ct;
    for (int i = s0; i < s1; ++i) {
        int8_t c = 3;
        if (i < n_cand) {
            const unsigned long long key = sel_key(pooled, i);
            if (key >= T1) {
                c = 2;
                imp_idx[ri++] = i;
            } else if (key >= T2) {
                c = 1;
                tbm_idx[rt++] = i;
            } else {
                c = 0;
            }
        }
        cls[i] = c;
    }
    if (tid == 0 && rank == 0) {
        int32_t* cnt = counts_all + 4 * u;
        cnt[0] = n_imp;
        cnt[1] = n_tbm;
        cnt[2] = n_cand - n_imp - n_tbm;
        cnt[3] = l_win;
    }
    cl_sync();  // no CTA exits while a peer may still read its shared memory
}

}  // namespace

cudaError_t launch_select(const Dims& dm, int l_win, int n_imp, int n_tbm, int kernel,
                          const float* glo, const float* loc, const ems_stage& sg,
                          DevStatus* status, cudaStream_t s, int policy, int sink, int n_budget) {
    static const int forced = [] {
        const char* e = getenv("EMS_SELECT_CLUSTER");  // A/B override: 0 never, 1 always
        return e ? atoi(e) : -1;
    }();
    // The cluster kernel pays for its cross-CTA exchanges with 8x the parallelism per unit:
    // worth it for long sequences when few units leave most SMs idle (config 3: 121 -> 35 us);
    // with many units the one-CTA-per-unit grid already fills the GPU (config 2: 20 vs 109 us).
    const bool auto_cluster = dm.L >= 8192 && (long long)dm.units * kClu <= 2 * 148;
    if ((forced < 0 ? auto_cluster : forced != 0) && dm.L >= 8 * kClu) {
        select_cluster_kernel<<<dm.units * kClu, kCThreads, 0, s>>>(
            glo, loc, dm.L, l_win, n_imp, n_tbm, kernel, sg.pooled, sg.cls, sg.imp_idx, sg.tbm_idx, sg.part_counts,
            dm.cap_c, dm.cap_tbm, status, dm.unit_base, policy, sink, n_budget);
        return cudaGetLastError();
    }
    select_kernel<<<dm.units, kSelThreads, 0, s>>>(glo, loc, dm.L, l_win, n_imp, n_tbm, kernel,
                                                   sg.pooled, sg.cls, sg.imp_idx, sg.tbm_idx,
                                                   sg.part_counts, dm.cap_c, dm.cap_tbm, status, dm.unit_base,
                                                   policy, sink, n_budget);
    return cudaGetLastError();
}

}  // namespace ems
