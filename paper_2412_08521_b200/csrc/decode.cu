// decode.cu -- (f2) the EMS decode step on the device: one CTA per KV unit,
// or, for small grids, a cluster of 8 CTAs per unit (see decode_step_kernel).
//
// Restates, per head (unit), decode_step (proj/src/engine.cpp:150-210):
//   append the raw (k, v) to the local window; expand the cache through its look-up table
//   (expand_cache, engine.cpp:84-132: every non-zero LUT entry materialises its center's
//   unit_key * key_norm RoPE'd at the entry's position (with_pos) or the center's
//   (without_pos), then the locals RoPE'd at their own positions); attend the RoPE'd query
//   over the expanded rows (attention_row_probs / weighted_value_sum); let the attention
//   mass flow back into the owning entries' glo and loc_cur; rotate the score windows every
//   l_win steps (cache.cpp:96-106); then decode_update (proj/src/compressor.cpp:376-398):
//   graduate the oldest locals beyond l_win into center slots (lowest free slot, LUT entry
//   appended, oldest zero-mapped / oldest LUT entry dropped at capacity) and, when the
//   centers exceed their capacity, retire the least important center
//   (retire_least_important_center, :286-372): merge it into its most redundant center
//   (R = cos(unit keys) * cos(values) >= tau, weights = combined Glo-Loc scores) or send its
//   LUT entries to the zero class / remove them.
// GQA (contract D2): the G query heads of a unit attend the same cache; the mass flowing
// back is the mean of their probabilities.
// Numerics: keys/values fp32, logits fp32 dot products, softmax exp in fp32 with an fp64
// normaliser, value sums in fp32 per warp slice combined in fp64, all score accumulators in
// fp64.  Every reduction runs in a fixed order (no float atomics) -> deterministic for a
// given launch shape.
#include <float.h>

#include "common.cuh"

namespace ems {

namespace {

// threads per CTA: 512 when there are few units (the per-unit phases are latency-bound, more
// warps per unit help), 256 when the grid already fills the SMs; reductions use the
// launched width, so results are a function of the problem shape only (deterministic)
constexpr int kTMax = 512;
constexpr int kWarpsMax = kTMax / 32;
constexpr int kDecClu = 8;  // CTAs per unit in the cluster variant

struct DecArgs {
    int G, d, S, W, T, R;          // query heads per unit; capacities: slots, locals, LUT, rows
    int l_win, cap_c, lut_cap;
    double tau;
    int zero_class, with_pos;
    long long position;
    int max_pos;
    const float2* table;           // [max_pos][d/2] (cos, sin)
    const void* q;                 // [units*G][d] raw
    const void* k;                 // [units][d] raw
    const void* v;                 // [units][d]
    int dtype;
    void* out;                     // [units*G][d]
    int32_t* argmax_pos;           // [units*G]
    ems_decode_state st;
    int32_t* row_owner;            // [units][R]
    int32_t* row_pos;              // [units][R]
    float* probs;                  // [units][G][R]
    float* pmean;                  // [units][R]
    int policy, sink, n_budget;    // ems_policy, PolicyHandle::sink_count, n_budget
};

__device__ __forceinline__ float ldx(const void* p, size_t i, int dtype) {
    return dtype == EMS_F32 ? static_cast<const float*>(p)[i]
                            : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ void stx(void* p, size_t i, int dtype, double x) {
    if (dtype == EMS_F32) static_cast<float*>(p)[i] = (float)x;
    else static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn((float)x);
}

// ---- block-wide helpers (fixed reduction order -> deterministic) ----------------------
__device__ double bsum(double v, double* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    __syncthreads();
    return t;
}
// (key, tie, idx) lexicographic "better" selection; better(a, b) decides.  Keys/ties are
// a total order on the candidates, so the result does not depend on reduction order.
struct Cand {
    double key;
    long long tie;
    int idx;
};
template <class Better>
__device__ Cand bselect(Cand c, Better better, Cand* sh) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Cand x;
        x.key = __shfl_xor_sync(0xffffffffu, c.key, o);
        x.tie = __shfl_xor_sync(0xffffffffu, c.tie, o);
        x.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
        if (better(x, c)) c = x;
    }
    __syncthreads();
    if (l == 0) sh[w] = c;
    __syncthreads();
    Cand t = sh[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
        if (better(sh[i], t)) t = sh[i];
    __syncthreads();
    return t;
}
// exclusive scan of one int per thread; returns the total in *tot
__device__ int bscan(int x, int* sh, int* tot) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (l >= o) inc += y;
    }
    __syncthreads();
    if (l == 31) sh[w] = inc;
    __syncthreads();
    int base = 0, all = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
        if (i < w) base += sh[i];
        all += sh[i];
    }
    __syncthreads();
    *tot = all;
    return base + inc - x;
}

// combined_entry_score, proj/src/compressor.cpp:261-267
__device__ __forceinline__ double combined(const double* sc, double align) {
    if (align <= 0.0) return sc[0];
    return fmax(sc[0] * align, sc[1] + sc[2]);
}

// kG: query heads per unit rounded up to a power of two (register arrays sized by it);
// kTh / kMinB: launch width and residency hint (512 x 1 for few units, 256 x 3 for many).
// kClu > 1: a unit's expanded rows are split over a cluster of kClu CTAs (row list, logits,
// softmax, value sums, argmax and the mass flow), with the cross-CTA maxima, normalisers,
// partial sums and per-owner masses exchanged through distributed shared memory in rank
// order; rank 0 then writes the cache alone, every rank scoring its slice of the centers in
// the retire step's redundancy pass.
template <int kG, int kTh, int kMinB, int kClu>
__global__ void __launch_bounds__(kTh, kMinB) decode_step_kernel(DecArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int rank = kClu > 1 ? (int)cl_rank() : 0;
    const int u = blockIdx.x / kClu, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kT = blockDim.x, kWarps = kT >> 5;
    const int d = a.d, S = a.S, W = a.W, T = a.T, G = a.G, pairs = d / 2;
    double* acc = reinterpret_cast<double*>(dsm);                  // [max(S + W, 8 d)] owner mass / R / partials
    float* qrot = reinterpret_cast<float*>(acc + max(S + W, kWarps * d));  // [G][d]
    double* vout = reinterpret_cast<double*>(qrot + ((G * d + 1) & ~1));   // [G][d] cluster partial outputs
    __shared__ int s_cnt;
    __shared__ float s_max[8];
    __shared__ double s_z[8];
    __shared__ Cand s_cand[8];
    __shared__ double shd[kWarpsMax];
    __shared__ Cand shc[kWarpsMax];
    __shared__ int shi[kWarpsMax];
    __shared__ int s_meta[8];
    __shared__ double s_w[4];
    __shared__ int s_i[4];

    const ems_decode_state& st = a.st;
    float* skey = st.slot_key + (size_t)u * S * d;
    float* snorm = st.slot_norm + (size_t)u * S;
    float* sval = st.slot_value + (size_t)u * S * d;
    int32_t* spos = st.slot_pos + (size_t)u * S;
    double* sscore = st.slot_score + (size_t)u * S * 3;
    int32_t* salive = st.slot_alive + (size_t)u * S;
    float* lkey = st.local_key + (size_t)u * W * d;
    float* lval = st.local_value + (size_t)u * W * d;
    int32_t* lpos = st.local_pos + (size_t)u * W;
    double* lscore = st.local_score + (size_t)u * W * 3;
    int32_t* tpos = st.lut_pos + (size_t)u * T;
    int32_t* tslot = st.lut_slot + (size_t)u * T;
    int32_t* meta = st.meta + (size_t)u * 8;
    int32_t* rown = a.row_owner + (size_t)u * a.R;
    int32_t* rpos = a.row_pos + (size_t)u * a.R;
    float* prob = a.probs + (size_t)u * G * a.R;
    float* pm = a.pmean + (size_t)u * a.R;

    if (tid < 8) s_meta[tid] = meta[tid];
    __syncthreads();
    int head = s_meta[0], count = s_meta[1], lut_n = s_meta[2];
    // Capacity guard: the step appends one local (ring of W) and expands at most lut_n + count + 1
    // rows (R).  A caller that steps past the horizon the state was sized for (max_positions)
    // gets EMS_CORRUPTION in meta[6] (ems_decode_sync_status) and the unit stops; every CTA of a
    // cluster reads the same meta, so they all leave here together.
    if (s_meta[6] != 0 || count + 1 > W || lut_n + count + 1 > a.R) {
        if (rank == 0 && tid == 0 && s_meta[6] == 0) meta[6] = EMS_CORRUPTION;
        return;
    }

    // 1. append the incoming token to the local window (engine.cpp:166-172)
    if (rank == 0) {
        const int slot = (head + count) % W;
        for (int i = tid; i < d; i += kT) {
            lkey[(size_t)slot * d + i] = ldx(a.k, (size_t)u * d + i, a.dtype);
            lval[(size_t)slot * d + i] = ldx(a.v, (size_t)u * d + i, a.dtype);
        }
        if (tid == 0) {
            lpos[slot] = (int32_t)a.position;
            lscore[3 * slot] = lscore[3 * slot + 1] = lscore[3 * slot + 2] = 0.0;
        }
    }
    ++count;
    if constexpr (kClu > 1) cl_sync();  // the appended row is read by other CTAs of the cluster
    else __syncthreads();               // ... or by another warp in step 3
    // 2. RoPE'd queries (apply_rope at the new position, engine.cpp:175)
    for (int x = tid; x < G * pairs; x += kT) {
        const int h = x / pairs, p = x % pairs;
        const float q0 = ldx(a.q, ((size_t)u * G + h) * d + 2 * p, a.dtype);
        const float q1 = ldx(a.q, ((size_t)u * G + h) * d + 2 * p + 1, a.dtype);
        const float2 cs = a.table[(size_t)a.position * pairs + p];
        qrot[h * d + 2 * p] = q0 * cs.x - q1 * cs.y;
        qrot[h * d + 2 * p + 1] = q0 * cs.y + q1 * cs.x;
    }
    // 3. expanded rows: non-zero LUT entries in LUT order, then the locals (expand_cache)
    int n_rows;
    if constexpr (kClu > 1) {  // rank r lists LUT slice r (offset = rows of the lower ranks) and locals slice r
        const int e0 = (int)((long long)rank * lut_n / kClu), e1 = (int)((long long)(rank + 1) * lut_n / kClu);
        int cnt = 0;
        for (int e = e0 + tid; e < e1; e += kT) cnt += tslot[e] >= 0;
        int tot;
        bscan(cnt, shi, &tot);
        if (tid == 0) s_cnt = tot;
        cl_sync();
        int base = 0, lut_rows = 0;
        for (int q = 0; q < kClu; ++q) {
            const int c = ld_dsm_i32(&s_cnt, q);
            base += q < rank ? c : 0;
            lut_rows += c;
        }
        for (int c0 = e0; c0 < e1; c0 += kT) {
            const int e = c0 + tid;
            const int keep = e < e1 && tslot[e] >= 0;
            const int off = bscan(keep, shi, &tot);
            if (keep) {
                rown[base + off] = tslot[e];
                rpos[base + off] = tpos[e];
            }
            base += tot;
        }
        const int l0 = rank * count / kClu, l1 = (rank + 1) * count / kClu;
        for (int li = l0 + tid; li < l1; li += kT) {
            const int ring = (head + li) % W;
            rown[lut_rows + li] = S + ring;
            rpos[lut_rows + li] = lpos[ring];
        }
        n_rows = lut_rows + count;
        cl_sync();  // the whole row list is visible to every CTA
    } else {
        int base = 0;
        for (int c0 = 0; c0 < lut_n; c0 += kT) {
            const int e = c0 + tid;
            const int keep = e < lut_n && tslot[e] >= 0;
            int tot;
            const int off = bscan(keep, shi, &tot);
            if (keep) {
                rown[base + off] = tslot[e];
                rpos[base + off] = tpos[e];
            }
            base += tot;
        }
        for (int li = tid; li < count; li += kT) {
            const int ring = (head + li) % W;
            rown[base + li] = S + ring;
            rpos[base + li] = lpos[ring];
        }
        n_rows = base + count;
        __syncthreads();
    }
    // this CTA's rows: [R0, R1) (all of them without a cluster)
    const int R0 = (int)((long long)rank * n_rows / kClu), R1 = (int)((long long)(rank + 1) * n_rows / kClu);
    // 4. logits: one warp per row, lanes over RoPE pairs; all G heads share the key.  The G
    //    (<= 8) per-lane partial dot products are reduced together in 9 shuffles (each step
    //    halves the values a lane carries), leaving head h's sum in lanes 4h' .. (fixed order).
    const float scale = rsqrtf((float)d);
    //    Few units (512-thread CTAs): two rows per warp pass, both rows' owners, norms, keys and
    //    RoPE factors loaded before either is used (the pass is latency-bound on L2); many
    //    units per SM (256 x 3) already overlap their loads and have no registers to spare.
    constexpr int kLR = kMinB > 1 ? 1 : 2;
    for (int r00 = R0 + warp; r00 < R1; r00 += kLR * kWarps) {
        int oo[kLR], rr[kLR];
#pragma unroll
        for (int t2 = 0; t2 < kLR; ++t2) {
            rr[t2] = r00 + t2 * kWarps;
            oo[t2] = rr[t2] < R1 ? rown[rr[t2]] : -1;
        }
        // d <= 128: at most two pairs per lane, all loaded before use (memory-level parallelism)
        float2 kk[kLR][2], cs[kLR][2];
        float kns[kLR];
#pragma unroll
        for (int t2 = 0; t2 < kLR; ++t2) {
            const int o = oo[t2], r = rr[t2];
            if (o < 0) continue;
            const bool center = o < S;
            const float* kb = center ? skey + (size_t)o * d : lkey + (size_t)(o - S) * d;
            kns[t2] = center ? snorm[o] : 1.f;
            const int rp = center && !a.with_pos ? spos[o] : rpos[r];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int p = lane + 32 * t;
                if (p < pairs) {
                    kk[t2][t] = reinterpret_cast<const float2*>(kb)[p];
                    cs[t2][t] = a.table[(size_t)rp * pairs + p];
                }
            }
        }
#pragma unroll
        for (int t2 = 0; t2 < kLR; ++t2) {
            const int r = rr[t2];
            if (oo[t2] < 0) continue;
            const float kn = kns[t2];
            float part[kG];
#pragma unroll
            for (int h = 0; h < kG; ++h) part[h] = 0.f;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int p = lane + 32 * t;
                if (p < pairs) {
                    const float k0 = kk[t2][t].x * kn, k1 = kk[t2][t].y * kn;
                    const float r0 = k0 * cs[t2][t].x - k1 * cs[t2][t].y, r1 = k0 * cs[t2][t].y + k1 * cs[t2][t].x;
#pragma unroll
                    for (int h = 0; h < kG; ++h)
                        if (h < G) {
                            const float2 qq = reinterpret_cast<const float2*>(qrot + h * d)[p];
                            part[h] += qq.x * r0 + qq.y * r1;
                        }
                }
            }
            // transpose-reduce: each xor-16, 8, ... step halves the values a lane carries (the lane
            // with the offset bit set keeps the upper half), so after log2(kG) steps lane L holds
            // head = its offset bits read from the top; the remaining xor steps finish that sum
            int h = 0, off = 16;
#pragma unroll
            for (int n = kG; n > 1; n >>= 1, off >>= 1) {
                const bool hi = lane & off;
#pragma unroll
                for (int i = 0; i < n / 2; ++i) {
                    const float send = hi ? part[i] : part[i + n / 2];
                    const float keep = hi ? part[i + n / 2] : part[i];
                    part[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                }
                h = 2 * h + (hi ? 1 : 0);
            }
            for (int o2 = off; o2 > 0; o2 >>= 1) part[0] += __shfl_xor_sync(0xffffffffu, part[0], o2);
            if ((lane & (2 * off - 1)) == 0 && h < G) prob[(size_t)h * a.R + r] = part[0] * scale;
        }
    }
    __syncthreads();
    // 5. softmax per query head (softmax_in_place: max-subtracted exp, fp64 normaliser), all
    //    heads per pass over this CTA's rows: per-head maxima, then fp64 normalisers (warp
    //    shuffles, warp partials combined in warp order; across a cluster in rank order)
    {
        __shared__ float s_wm[kWarpsMax][8];
        __shared__ double s_wz[kWarpsMax][8];
        float mh[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) mh[h] = -FLT_MAX;
        for (int r = R0 + tid; r < R1; r += kT)
#pragma unroll
            for (int h = 0; h < kG; ++h)
                if (h < G) mh[h] = fmaxf(mh[h], prob[(size_t)h * a.R + r]);
#pragma unroll
        for (int h = 0; h < kG; ++h) {
            mh[h] = warp_max(mh[h]);
            if (lane == 0) s_wm[warp][h] = mh[h];
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kG; ++h) {
            float m = -FLT_MAX;
            for (int w2 = 0; w2 < kWarps; ++w2) m = fmaxf(m, s_wm[w2][h]);
            mh[h] = m;
        }
        if constexpr (kClu > 1) {  // cluster-wide max
            if (tid < G) s_max[tid] = mh[tid];
            cl_sync();
#pragma unroll
            for (int h = 0; h < kG; ++h) {
                float m = -FLT_MAX;
                if (h < G)
                    for (int q = 0; q < kClu; ++q) m = fmaxf(m, ld_dsm_f32(&s_max[h], q));
                mh[h] = m;
            }
        }
        double zh[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) zh[h] = 0.0;
        for (int r = R0 + tid; r < R1; r += kT)
#pragma unroll
            for (int h = 0; h < kG; ++h)
                if (h < G) zh[h] += (double)expf(prob[(size_t)h * a.R + r] - mh[h]);
#pragma unroll
        for (int h = 0; h < kG; ++h) {
            zh[h] = warp_sum(zh[h]);
            if (lane == 0) s_wz[warp][h] = zh[h];
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < kG; ++h) {
            double z = 0.0;
            for (int w2 = 0; w2 < kWarps; ++w2) z += s_wz[w2][h];
            zh[h] = z;
        }
        if constexpr (kClu > 1) {  // normalisers summed in rank order
            if (tid < G) s_z[tid] = zh[tid];
            cl_sync();
#pragma unroll
            for (int h = 0; h < kG; ++h) {
                double z = 0.0;
                if (h < G)
                    for (int q = 0; q < kClu; ++q) z += ld_dsm_f64(&s_z[h], q);
                zh[h] = z;
            }
        }
        for (int r = R0 + tid; r < R1; r += kT)
#pragma unroll
            for (int h = 0; h < kG; ++h)
                if (h < G) {
                    float* ph = prob + (size_t)h * a.R;
                    ph[r] = (float)((double)expf(ph[r] - mh[h]) / zh[h]);
                }
        __syncthreads();
    }
    // 6. outputs (weighted_value_sum): warp w sums a contiguous block of rows (in order) for all
    //    G heads at once in fp32 (each value row is read once), lanes over d; the warp partials
    //    combine in warp order in fp64, one head at a time.
    {
        const int per = (R1 - R0 + kWarps - 1) / kWarps;
        const int r0 = min(R1, R0 + warp * per), r1 = min(R1, r0 + per);
        const int epl = (d + 31) / 32;  // elements per lane (d <= 128 -> <= 4)
        double* part = acc;              // [kWarps][d] for one head at a time (acc is free here)
        float o[kG][4];
#pragma unroll
        for (int h = 0; h < kG; ++h)
#pragma unroll
            for (int e = 0; e < 4; ++e) o[h][e] = 0.f;
        constexpr int kU = 4;  // rows in flight per warp (their value loads issued together)
        for (int rb = r0; rb < r1; rb += kU) {
            float vv[kU][4];
#pragma unroll
            for (int t = 0; t < kU; ++t) {
                const int r = rb + t;
                const int ow = r < r1 ? rown[r] : 0;
                const float* vr = ow < S ? sval + (size_t)ow * d : lval + (size_t)(ow - S) * d;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    vv[t][e] = (r < r1 && e < epl && lane * epl + e < d) ? vr[lane * epl + e] : 0.f;
            }
#pragma unroll
            for (int t = 0; t < kU; ++t) {
                const int r = rb + t;
                if (r >= r1) break;
#pragma unroll
                for (int h = 0; h < kG; ++h)
                    if (h < G) {
                        const float p = prob[(size_t)h * a.R + r];
#pragma unroll
                        for (int e = 0; e < 4; ++e) o[h][e] = fmaf(p, vv[t][e], o[h][e]);
                    }
            }
        }
#pragma unroll
        for (int h = 0; h < kG; ++h) {
            if (h >= G) break;
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (e < epl && lane * epl + e < d) part[warp * d + lane * epl + e] = (double)o[h][e];
            __syncthreads();
            for (int i = tid; i < d; i += kT) {
                double t = 0.0;
                for (int w2 = 0; w2 < kWarps; ++w2) t += part[w2 * d + i];
                if constexpr (kClu > 1) vout[h * d + i] = t;
                else stx(a.out, ((size_t)u * G + h) * d + i, a.dtype, t);
            }
        }
        __syncthreads();
        if constexpr (kClu > 1) {  // the CTAs' partial outputs, summed in rank order
            cl_sync();
            for (int x = rank * kT + tid; x < G * d; x += kClu * kT) {
                double t = 0.0;
                for (int q = 0; q < kClu; ++q) t += ld_dsm_f64(&vout[x], q);
                stx(a.out, (size_t)u * G * d + x, a.dtype, t);
            }
        }
    }
    auto better = [](const Cand& x, const Cand& y) {
        if (y.idx < 0) return x.idx >= 0;
        if (x.idx < 0) return false;
        return x.key > y.key || (x.key == y.key && x.tie < y.tie);  // first max (engine.cpp:188-191)
    };
    // 7. argmax per head (first max) and 8a. the GQA-mean probability per row, one pass over
    //    the rows for all heads; per-head candidates reduced by warp shuffles, then across warps
    //    in warp order by warp 0
    {
        float ck[kG];
        int ci[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) ck[h] = -1.f, ci[h] = -1;
        for (int r = R0 + tid; r < R1; r += kT) {
            double sum = 0.0;
#pragma unroll
            for (int h = 0; h < kG; ++h)
                if (h < G) {
                    const float p = prob[(size_t)h * a.R + r];
                    sum += (double)p;
                    if (ci[h] < 0 || p > ck[h]) ck[h] = p, ci[h] = r;
                }
            pm[r] = (float)(sum / G);
        }
#pragma unroll
        for (int h = 0; h < kG; ++h)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ok = __shfl_xor_sync(0xffffffffu, ck[h], o);
                const int oi = __shfl_xor_sync(0xffffffffu, ci[h], o);
                if (oi >= 0 && (ci[h] < 0 || ok > ck[h] || (ok == ck[h] && oi < ci[h]))) ck[h] = ok, ci[h] = oi;
            }
        __shared__ float s_ak[kWarpsMax][8];
        __shared__ int s_ai[kWarpsMax][8];
        if (lane == 0)
#pragma unroll
            for (int h = 0; h < kG; ++h) s_ak[warp][h] = ck[h], s_ai[warp][h] = ci[h];
        __syncthreads();
        if (warp == 0 && lane < G) {
            float bk = -1.f;
            int bi = -1;
            for (int w2 = 0; w2 < kWarps; ++w2) {
                const float ok = s_ak[w2][lane];
                const int oi = s_ai[w2][lane];
                if (oi >= 0 && (bi < 0 || ok > bk || (ok == bk && oi < bi))) bk = ok, bi = oi;
            }
            if constexpr (kClu > 1) s_cand[lane] = Cand{(double)bk, bi, bi};
            else a.argmax_pos[(size_t)u * G + lane] = bi >= 0 ? rpos[bi] : -1;
        }
    }
    if constexpr (kClu > 1) {  // candidates of the CTAs (global row indices: a total order)
        cl_sync();
        if (rank == 0 && tid < G) {
            Cand c{-1.0, 0, -1};
            for (int q = 0; q < kClu; ++q) {
                const Cand x{ld_dsm_f64(&s_cand[tid].key, q), ld_dsm_i64(&s_cand[tid].tie, q),
                             ld_dsm_i32(&s_cand[tid].idx, q)};
                if (better(x, c)) c = x;
            }
            a.argmax_pos[(size_t)u * G + tid] = c.idx >= 0 ? rpos[c.idx] : -1;
        }
    }
    for (int i = tid; i < S + W; i += kT) acc[i] = 0.0;
    __syncthreads();
    // ordered pass: rows in order, equal owners inside a 32-row chunk summed in lane order
    if constexpr (kClu > 1) {
        // a few hundred rows per CTA: warp 0 alone, four chunks' owners and masses loaded
        // before the first is summed (fewer block barriers than the round scheme below)
        constexpr int kOP = 4;
        if (warp == 0)
            for (int b0 = R0; b0 < R1; b0 += kOP * 32) {
                int oc[kOP];
                double pc[kOP];
#pragma unroll
                for (int t = 0; t < kOP; ++t) {
                    const int r = b0 + 32 * t + lane;
                    oc[t] = r < R1 ? rown[r] : -1 - lane;
                    pc[t] = r < R1 ? (G == 1 ? (double)prob[r] : (double)pm[r]) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < kOP; ++t) {
                    if (b0 + 32 * t >= R1) break;
                    const int r = b0 + 32 * t + lane, o = oc[t];
                    const unsigned grp = __match_any_sync(0xffffffffu, o);
                    double gs = 0.0;
                    for (unsigned m = grp; m; m &= m - 1) gs += __shfl_sync(grp, pc[t], __ffs(m) - 1);
                    if (r < R1 && lane == __ffs(grp) - 1) acc[o] += gs;
                    __syncwarp();
                }
            }
    } else {
        // all of a unit's rows in one CTA: each round, warp w forms the group sums of chunk
        // (round, w) (match + lane-order shuffles, every warp in parallel); warp 0 then adds
        // the round's chunks into acc in chunk order (a chunk's group leaders have distinct
        // owners, so its lanes add at once) -- the same sums in the same order as above
        __shared__ int s_go[kWarpsMax][32];
        __shared__ double s_gs[kWarpsMax][32];
        for (int b0 = R0; b0 < R1; b0 += kWarps * 32) {
            const int r = b0 + 32 * warp + lane;
            const int o = r < R1 ? rown[r] : -1 - lane;
            const double p = r < R1 ? (G == 1 ? (double)prob[r] : (double)pm[r]) : 0.0;
            const unsigned grp = __match_any_sync(0xffffffffu, o);
            double gs = 0.0;
            for (unsigned m = grp; m; m &= m - 1) gs += __shfl_sync(grp, p, __ffs(m) - 1);
            s_go[warp][lane] = r < R1 && lane == __ffs(grp) - 1 ? o : -1;
            s_gs[warp][lane] = gs;
            __syncthreads();
            if (warp == 0)
                for (int w2 = 0; w2 < kWarps && b0 + 32 * w2 < R1; ++w2) {
                    const int ow = s_go[w2][lane];
                    if (ow >= 0) acc[ow] += s_gs[w2][lane];
                    __syncwarp();
                }
            __syncthreads();
        }
    }
    __syncthreads();
    if constexpr (kClu > 1) {  // owners split over the CTAs; each owner's mass summed in rank order
        cl_sync();
        const int o0 = (int)((long long)rank * (S + W) / kClu), o1 = (int)((long long)(rank + 1) * (S + W) / kClu);
        for (int o = o0 + tid; o < o1; o += kT) {
            double t = 0.0;
            for (int q = 0; q < kClu; ++q) t += ld_dsm_f64(&acc[o], q);
            if (o < S) {
                if (salive[o]) sscore[3 * o] += t, sscore[3 * o + 2] += t;
            } else if ((o - S - head + W) % W < count) {  // a live local
                lscore[3 * (o - S)] += t;
                lscore[3 * (o - S) + 2] += t;
            }
        }
        cl_sync();  // every score update visible, every remote read done
    } else {
        for (int s = tid; s < S; s += kT)
            if (salive[s]) sscore[3 * s] += acc[s], sscore[3 * s + 2] += acc[s];
        for (int li = tid; li < count; li += kT) {
            const int ring = (head + li) % W;
            lscore[3 * ring] += acc[S + ring];
            lscore[3 * ring + 2] += acc[S + ring];
        }
    }
    // 9. score window rotation every l_win steps (engine.cpp:196-200)
    int wfill = s_meta[3] + 1;
    if (wfill >= a.l_win) {
        if (rank == 0) {
            for (int s = tid; s < S; s += kT)
                if (salive[s]) sscore[3 * s + 1] = sscore[3 * s + 2], sscore[3 * s + 2] = 0.0;
            for (int li = tid; li < count; li += kT) {
                const int ring = (head + li) % W;
                lscore[3 * ring + 1] = lscore[3 * ring + 2];
                lscore[3 * ring + 2] = 0.0;
            }
        }
        wfill = 0;
    }
    __syncthreads();
    // 10. policy_decode_compress (policies.cpp:182-242): EMS decode_update (compressor.cpp:376-398);
    //     SnapKV / H2O / StreamingLLM graduate_locals (policies.cpp:88-98) then drop; full: identity.
    //     With a cluster, rank 0 alone writes the cache; every rank takes part in the retire
    //     step's redundancy pass (its slice of the centers, candidates gathered in rank order).
    int n_alive = s_meta[5], compressed = s_meta[4];
    const bool ems = a.policy == EMS_POLICY_EMS;
    while (a.policy != EMS_POLICY_FULL && count > a.l_win) {
        const int g = head;  // graduating local (front of the window)
        // 10a. oldest zero-mapped (else oldest) LUT entry leaves at capacity (:272-284)
        if (rank == 0 && ems && lut_n >= a.lut_cap) {
            Cand c{0.0, 0, -1};
            for (int e = tid; e < lut_n; e += kT)
                if (tslot[e] < 0 && (c.idx < 0 || e < c.idx)) c = Cand{0.0, e, e};
            auto first = [](const Cand& x, const Cand& y) {
                return x.idx >= 0 && (y.idx < 0 || x.idx < y.idx);
            };
            c = bselect(c, first, shc);
            const int at = c.idx >= 0 ? c.idx : 0;
            for (int c0 = at + 1; c0 < lut_n; c0 += kT) {
                const int e = c0 + tid;
                int pp = 0, ss = 0;
                if (e < lut_n) pp = tpos[e], ss = tslot[e];
                __syncthreads();
                if (e < lut_n) tpos[e - 1] = pp, tslot[e - 1] = ss;
                __syncthreads();
            }
            --lut_n;
        }
        // 10b. insert_center: lowest free slot (cache.cpp:48-57)
        if (rank == 0) {
            Cand fs{0.0, 0, -1};
            for (int s = tid; s < S; s += kT)
                if (!salive[s] && (fs.idx < 0 || s < fs.idx)) fs = Cand{0.0, s, s};
            auto lower = [](const Cand& x, const Cand& y) { return x.idx >= 0 && (y.idx < 0 || x.idx < y.idx); };
            fs = bselect(fs, lower, shc);
            const int slot = fs.idx >= 0 ? fs.idx : 0;  // no free slot: corrupt state, recorded below
            if (fs.idx < 0 && tid == 0) meta[6] = EMS_CORRUPTION;
            double kk = 0.0;
            for (int i = tid; i < d; i += kT) kk += (double)lkey[(size_t)g * d + i] * lkey[(size_t)g * d + i];
            const double kn = sqrt(bsum(kk, shd));  // normalized_or_zero, :16-25
            for (int i = tid; i < d; i += kT) {
                const float x = lkey[(size_t)g * d + i];
                skey[(size_t)slot * d + i] = kn > 0.0 ? (float)((double)x / kn) : x;
                sval[(size_t)slot * d + i] = lval[(size_t)g * d + i];
            }
            if (tid == 0) {
                snorm[slot] = (float)kn;
                spos[slot] = lpos[g];
                for (int t = 0; t < 3; ++t) sscore[3 * slot + t] = lscore[3 * g + t];
                salive[slot] = 1;
                tpos[lut_n] = lpos[g];
                tslot[lut_n] = slot;
            }
        }
        ++lut_n;
        ++n_alive;
        head = (head + 1) % W;
        --count;
        __syncthreads();
        if (!ems || n_alive <= a.cap_c) continue;
        if constexpr (kClu > 1) cl_sync();  // rank 0's insert and window rotation visible to every rank
        // 10c. retire_least_important_center (:286-372)
        double sg = 0.0, sl = 0.0;
        for (int s = tid; s < S; s += kT)
            if (salive[s]) sg += sscore[3 * s], sl += sscore[3 * s + 1] + sscore[3 * s + 2];
        for (int li = tid; li < count; li += kT) {
            const int ring = (head + li) % W;
            sg += lscore[3 * ring];
            sl += lscore[3 * ring + 1] + lscore[3 * ring + 2];
        }
        sg = bsum(sg, shd);
        sl = bsum(sl, shd);
        const double align = sg > 0.0 ? sl / sg : 0.0;  // alignment_ratio, :244-259
        Cand tb{0.0, 0, -1};
        for (int s = tid; s < S; s += kT)
            if (salive[s]) {
                const Cand x{combined(sscore + 3 * s, align), spos[s], s};
                if (tb.idx < 0 || x.key < tb.key || (x.key == tb.key && x.tie < tb.tie)) tb = x;
            }
        auto least = [](const Cand& x, const Cand& y) {
            if (y.idx < 0) return x.idx >= 0;
            if (x.idx < 0) return false;
            return x.key < y.key || (x.key == y.key && x.tie < y.tie);
        };
        tb = bselect(tb, least, shc);
        const int ts = tb.idx;
        // R(tbm, c) for every other alive center: one warp per center; lane owns elements
        // [4 lane, 4 lane + 4) (d <= 128, d % 4 == 0), the retiring center stays in registers.
        // kRU centers per warp pass: their alive flags, norms, keys and values are all loaded
        // before the first is used (the pass is latency-bound on L2, one CTA per unit)
        constexpr int kRU = kMinB > 1 ? 1 : 4;
        double vv = 0.0;
        for (int i = tid; i < d; i += kT) vv += (double)sval[(size_t)ts * d + i] * sval[(size_t)ts * d + i];
        const double nv1 = sqrt(bsum(vv, shd));
        const float tnorm = snorm[ts];
        const bool act = 4 * lane < d;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 kt4 = act ? reinterpret_cast<const float4*>(skey + (size_t)ts * d)[lane] : z4;
        const float4 vt4 = act ? reinterpret_cast<const float4*>(sval + (size_t)ts * d)[lane] : z4;
        const int c_lo = (int)((long long)rank * S / kClu), c_hi = (int)((long long)(rank + 1) * S / kClu);
        for (int c0 = c_lo + warp; c0 < c_hi; c0 += kRU * kWarps) {
            float4 kcs[kRU], vcs[kRU];
            int alv[kRU];
            float cns[kRU];
#pragma unroll
            for (int t = 0; t < kRU; ++t) {
                const int c = c0 + t * kWarps;
                const bool in = c < c_hi;
                alv[t] = in ? salive[c] : 0;
                cns[t] = in ? snorm[c] : 0.f;
                kcs[t] = in && act ? reinterpret_cast<const float4*>(skey + (size_t)c * d)[lane] : z4;
                vcs[t] = in && act ? reinterpret_cast<const float4*>(sval + (size_t)c * d)[lane] : z4;
            }
#pragma unroll
            for (int t = 0; t < kRU; ++t) {
                const int c = c0 + t * kWarps;
                if (!alv[t] || c == ts) continue;
                const float4 kc = kcs[t], vc = vcs[t];
                double p0 = (double)kt4.x * kc.x + (double)kt4.y * kc.y + (double)kt4.z * kc.z + (double)kt4.w * kc.w;
                double p1 = (double)vt4.x * vc.x + (double)vt4.y * vc.y + (double)vt4.z * vc.z + (double)vt4.w * vc.w;
                double p2 = (double)vc.x * vc.x + (double)vc.y * vc.y + (double)vc.z * vc.z + (double)vc.w * vc.w;
                // transpose-reduce {kd, vd, v2, 0}: xor-16 and xor-8 halve the values a lane carries
                // (lanes 0-7 end with kd, 8-15 vd, 16-23 v2), xor-4/2/1 finish each sum
                {
                    const bool h16 = lane & 16, h8 = lane & 8;
                    const double k0 = h16 ? p2 : p0, k1 = h16 ? 0.0 : p1;
                    const double s0 = h16 ? p0 : p2, s1 = h16 ? p1 : 0.0;
                    const double b0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 16);
                    const double b1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 16);
                    double cacc = (h8 ? b1 : b0) + __shfl_xor_sync(0xffffffffu, h8 ? b0 : b1, 8);
                    cacc += __shfl_xor_sync(0xffffffffu, cacc, 4);
                    cacc += __shfl_xor_sync(0xffffffffu, cacc, 2);
                    cacc += __shfl_xor_sync(0xffffffffu, cacc, 1);
                    p0 = __shfl_sync(0xffffffffu, cacc, 0);
                    p1 = __shfl_sync(0xffffffffu, cacc, 8);
                    p2 = __shfl_sync(0xffffffffu, cacc, 16);
                }
                const double kd = p0, vd = p1, v2 = p2;
                if (lane == 0) {
                    double r = 0.0;
                    if (tnorm > 0.f && cns[t] > 0.f) {
                        const double ck = fmin(fmax(kd, -1.0), 1.0);
                        const double nv2 = sqrt(v2);
                        const double cv = (nv1 > 0.0 && nv2 > 0.0) ? fmin(fmax(vd / (nv1 * nv2), -1.0), 1.0) : 0.0;
                        r = ck * cv;
                    }
                    acc[c] = r;
                }
            }
        }
        __syncthreads();
        Cand bs{0.0, 0, -1};
        for (int c = c_lo + tid; c < c_hi; c += kT)
            if (salive[c] && c != ts) {
                const Cand x{acc[c], spos[c], c};
                if (bs.idx < 0 || x.key > bs.key || (x.key == bs.key && x.tie < bs.tie)) bs = x;
            }
        auto most = [](const Cand& x, const Cand& y) {
            if (y.idx < 0) return x.idx >= 0;
            if (x.idx < 0) return false;
            return x.key > y.key || (x.key == y.key && x.tie < y.tie);
        };
        bs = bselect(bs, most, shc);
        if constexpr (kClu > 1) {  // the ranks' candidates into rank 0, reduced in rank order
            __shared__ Cand s_rc[kClu];
            if (tid == 0) {
                st_dsm_f64(&s_rc[rank].key, 0, bs.key);
                st_dsm_i64(&s_rc[rank].tie, 0, bs.tie);
                st_dsm_i32(&s_rc[rank].idx, 0, bs.idx);
            }
            cl_sync();
            if (rank == 0) {
                bs = Cand{0.0, 0, -1};
                for (int q = 0; q < kClu; ++q)
                    if (most(s_rc[q], bs)) bs = s_rc[q];
            }
        }
        const int best = bs.idx;
        // only rank 0 writes the cache
        if (rank == 0 && best >= 0 && bs.key >= a.tau) {  // merge into the most redundant center
            if (tid == 0) {
                double wd = combined(sscore + 3 * best, align), wt = combined(sscore + 3 * ts, align);
                double ws = wd + wt;
                if (ws <= 0.0) wd = 0.5, wt = 0.5, ws = 1.0;
                s_w[0] = wd / ws;
                s_w[1] = wt / ws;
            }
            __syncthreads();
            const double fd = s_w[0], ft = s_w[1];
            double mk2 = 0.0;
            for (int i = tid; i < d; i += kT) {
                const double m = fd * skey[(size_t)best * d + i] + ft * skey[(size_t)ts * d + i];
                mk2 += m * m;
            }
            const double mn = sqrt(bsum(mk2, shd));
            for (int i = tid; i < d; i += kT) {
                const double m = fd * skey[(size_t)best * d + i] + ft * skey[(size_t)ts * d + i];
                const double mv = fd * sval[(size_t)best * d + i] + ft * sval[(size_t)ts * d + i];
                if (mn > 0.0) skey[(size_t)best * d + i] = (float)(m / mn);
                sval[(size_t)best * d + i] = (float)mv;
            }
            if (tid == 0)
                for (int t = 0; t < 3; ++t) sscore[3 * best + t] += sscore[3 * ts + t];
            for (int e = tid; e < lut_n; e += kT)
                if (tslot[e] == ts) tslot[e] = best;
        } else if (rank == 0 && a.zero_class) {
            for (int e = tid; e < lut_n; e += kT)
                if (tslot[e] == ts) tslot[e] = -1;
        } else if (rank == 0) {  // explicit removal: stable in-place compaction of the LUT
            int base = 0;
            for (int c0 = 0; c0 < lut_n; c0 += kT) {
                const int e = c0 + tid;
                int pp = 0, ss = 0;
                const int keep = e < lut_n && tslot[e] != ts;
                if (e < lut_n) pp = tpos[e], ss = tslot[e];
                int tot;
                const int off = bscan(keep, shi, &tot);
                if (keep) tpos[base + off] = pp, tslot[base + off] = ss;
                base += tot;
                __syncthreads();
            }
            lut_n = base;
        }
        __syncthreads();
        if (tid == 0 && rank == 0) salive[ts] = 0;
        --n_alive;
        compressed = 1;
        __syncthreads();
    }
    if (rank != 0) return;
    // 10d. H2O: drop the lowest-glo centers beyond capacity (ties -> lower position);
    //      StreamingLLM: drop the oldest non-sink center while over budget (policies.cpp:200-241)
    while ((a.policy == EMS_POLICY_H2O && n_alive > a.cap_c) ||
           (a.policy == EMS_POLICY_STREAMING && n_alive + count > a.n_budget)) {
        Cand w{0.0, 0, -1};
        for (int s = tid; s < S; s += kT)
            if (salive[s]) {
                Cand x;
                if (a.policy == EMS_POLICY_H2O) x = Cand{sscore[3 * s], spos[s], s};
                else if (spos[s] >= a.sink) x = Cand{(double)spos[s], spos[s], s};
                else continue;
                if (w.idx < 0 || x.key < w.key || (x.key == w.key && x.tie < w.tie)) w = x;
            }
        auto least2 = [](const Cand& x, const Cand& y) {
            if (y.idx < 0) return x.idx >= 0;
            if (x.idx < 0) return false;
            return x.key < y.key || (x.key == y.key && x.tie < y.tie);
        };
        w = bselect(w, least2, shc);
        if (w.idx < 0) break;  // nothing evictable
        const int ds_ = w.idx;
        // drop_center (policies.cpp:100-106): erase its LUT entries (stable), free the slot
        int base = 0;
        for (int c0 = 0; c0 < lut_n; c0 += kT) {
            const int e = c0 + tid;
            int pp = 0, ss = 0;
            const int keep = e < lut_n && tslot[e] != ds_;
            if (e < lut_n) pp = tpos[e], ss = tslot[e];
            int tot;
            const int off = bscan(keep, shi, &tot);
            if (keep) tpos[base + off] = pp, tslot[base + off] = ss;
            base += tot;
            __syncthreads();
        }
        lut_n = base;
        if (tid == 0) salive[ds_] = 0;
        --n_alive;
        compressed = 1;
        __syncthreads();
    }
    if (tid == 0) {
        meta[0] = head;
        meta[1] = count;
        meta[2] = lut_n;
        meta[3] = wfill;
        meta[4] = compressed;
        meta[5] = n_alive;
    }
}

// Decode state from a prefill cache (policy_prefill_compress output, slots in order).
template <typename T>
__global__ void decode_init_kernel(ems_cache c, ems_decode_state st, int d, int cap_c, int cap_l, int cap_lut,
                                   int S, int W, int T_) {
    const int u = blockIdx.x, tid = threadIdx.x;
    const int32_t* cnt = c.counts + 4 * u;
    const int nc = cnt[0], nl = cnt[1], nu = cnt[2];
    const T* ck = static_cast<const T*>(c.center_key) + (size_t)u * cap_c * d;
    const T* cv = static_cast<const T*>(c.center_value) + (size_t)u * cap_c * d;
    const T* lk = static_cast<const T*>(c.local_key) + (size_t)u * cap_l * d;
    const T* lv = static_cast<const T*>(c.local_value) + (size_t)u * cap_l * d;
    for (int x = tid; x < S * d; x += blockDim.x) {
        const int s = x / d;
        st.slot_key[(size_t)u * S * d + x] = s < nc ? ld(ck + x) : 0.f;
        st.slot_value[(size_t)u * S * d + x] = s < nc ? ld(cv + x) : 0.f;
    }
    for (int s = tid; s < S; s += blockDim.x) {
        st.slot_alive[(size_t)u * S + s] = s < nc;
        st.slot_norm[(size_t)u * S + s] = s < nc ? c.center_norm[(size_t)u * cap_c + s] : 0.f;
        st.slot_pos[(size_t)u * S + s] = s < nc ? c.center_pos[(size_t)u * cap_c + s] : 0;
        for (int t = 0; t < 3; ++t)
            st.slot_score[((size_t)u * S + s) * 3 + t] = s < nc ? c.center_score[((size_t)u * cap_c + s) * 3 + t] : 0.0;
    }
    for (int x = tid; x < W * d; x += blockDim.x) {
        const int l = x / d;
        st.local_key[(size_t)u * W * d + x] = l < nl ? ld(lk + x) : 0.f;
        st.local_value[(size_t)u * W * d + x] = l < nl ? ld(lv + x) : 0.f;
    }
    for (int l = tid; l < W; l += blockDim.x) {
        st.local_pos[(size_t)u * W + l] = l < nl ? c.local_pos[(size_t)u * cap_l + l] : 0;
        for (int t = 0; t < 3; ++t)
            st.local_score[((size_t)u * W + l) * 3 + t] = l < nl ? c.local_score[((size_t)u * cap_l + l) * 3 + t] : 0.0;
    }
    for (int e = tid; e < T_; e += blockDim.x) {
        st.lut_pos[(size_t)u * T_ + e] = e < nu ? c.lut_pos[(size_t)u * cap_lut + e] : 0;
        st.lut_slot[(size_t)u * T_ + e] = e < nu ? c.lut_slot[(size_t)u * cap_lut + e] : 0;
    }
    if (tid == 0) {
        int32_t* m = st.meta + 8 * u;
        m[0] = 0;        // ring head
        m[1] = nl;       // locals
        m[2] = nu;       // LUT entries
        m[3] = 0;        // window_fill (engine.cpp:74)
        m[4] = cnt[3];   // compressed
        m[5] = nc;       // alive centers
        m[6] = m[7] = 0;
    }
}

// RoPE table: (cos, sin) of pos * base^(-2i/d) in fp64, rounded to fp32 (rope.cpp:17-26)
__global__ void rope_table_kernel(float2* t, int max_pos, int pairs, int d, double base) {
    const size_t n = (size_t)max_pos * pairs;
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(x % pairs);
        const long long pos = (long long)(x / pairs);
        const double ang = (double)pos * pow(base, -(double)(2 * p) / (double)d);
        double s, c;
        sincos(ang, &s, &c);
        t[x] = make_float2((float)c, (float)s);
    }
}

}  // namespace

cudaError_t launch_rope_table(float2* table, int max_pos, int d, double base, cudaStream_t s) {
    rope_table_kernel<<<4 * 148, 256, 0, s>>>(table, max_pos, d / 2, d, base);
    return cudaGetLastError();
}

cudaError_t launch_decode_init(const Dims& m, int dtype, const ems_cache& c, const ems_decode_state& st,
                               int S, int W, int T, cudaStream_t s) {
    if (dtype == EMS_F32)
        decode_init_kernel<float><<<m.units, 256, 0, s>>>(c, st, m.d, m.cap_c, m.cap_l, m.cap_lut, S, W, T);
    else
        decode_init_kernel<__nv_bfloat16><<<m.units, 256, 0, s>>>(c, st, m.d, m.cap_c, m.cap_l, m.cap_lut, S, W,
                                                                  T);
    return cudaGetLastError();
}

cudaError_t launch_decode_step(const Dims& m, int dtype, int S, int W, int T, int R, int l_win, int lut_cap,
                               double tau, int zero_class, int with_pos, long long position, int max_pos,
                               const float2* table, const void* q, const void* k, const void* v, void* out,
                               int32_t* argmax_pos, const ems_decode_state& st, void* ws, cudaStream_t s,
                               int policy, int sink, int n_budget) {
    DecArgs a;
    a.policy = policy;
    a.sink = sink;
    a.n_budget = n_budget;
    a.G = m.G;
    a.d = m.d;
    a.S = S;
    a.W = W;
    a.T = T;
    a.R = R;
    a.l_win = l_win;
    a.cap_c = m.cap_c;
    a.lut_cap = lut_cap;
    a.tau = tau;
    a.zero_class = zero_class;
    a.with_pos = with_pos;
    a.position = position;
    a.max_pos = max_pos;
    a.table = table;
    a.q = q;
    a.k = k;
    a.v = v;
    a.dtype = dtype;
    a.out = out;
    a.argmax_pos = argmax_pos;
    a.st = st;
    char* p = static_cast<char*>(ws);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) / 256 * 256;
        return r;
    };
    const size_t U = m.units;
    a.row_owner = reinterpret_cast<int32_t*>(take(U * R * 4));
    a.row_pos = reinterpret_cast<int32_t*>(take(U * R * 4));
    a.probs = reinterpret_cast<float*>(take(U * m.G * R * 4));
    a.pmean = reinterpret_cast<float*>(take(U * R * 4));
    const bool wide = m.units < 148;  // few units: more warps per unit; many: more units per SM
    // a unit split over a cluster of kDecClu CTAs when the grid is small and the rows many
    static const int force_clu = [] {
        const char* e = getenv("EMS_DECODE_CLUSTER");  // 0 never, 1 always (A/B, tests)
        return e ? atoi(e) : -1;
    }();
    const bool clu = force_clu >= 0 ? force_clu == 1 : m.units * kDecClu <= 2 * 148;
    const int threads = wide || clu ? kTMax : 256;
    const size_t smem =
        (size_t)max(S + W, (threads / 32) * m.d) * 8 + (size_t)((m.G * m.d + 1) & ~1) * 4 + (size_t)m.G * m.d * 8;
    const int gb = m.G <= 1 ? 1 : m.G <= 2 ? 2 : m.G <= 4 ? 4 : 8;
    void (*fn)(DecArgs) = nullptr;
#define EMS_DEC_PICK(K)                                                                                   \
    if (gb == K)                                                                                          \
        fn = clu ? decode_step_kernel<K, kTMax, 1, kDecClu>                                               \
                 : (wide ? decode_step_kernel<K, kTMax, 1, 1> : decode_step_kernel<K, 256, 3, 1>);
    EMS_DEC_PICK(1) EMS_DEC_PICK(2) EMS_DEC_PICK(4) EMS_DEC_PICK(8)
#undef EMS_DEC_PICK
    if (!fn || m.G > 8) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) {
        const cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn), (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (!clu) {
        fn<<<m.units, threads, smem, s>>>(a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(m.units * kDecClu);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDecClu;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, a);
}

// Dynamic shared memory of the decode step (the largest launch variant): the per-owner mass /
// redundancy accumulator over S slots + W locals, the RoPE'd queries and the cluster partials.
size_t decode_smem_bytes(const Dims& m, int S, int W) {
    const size_t acc = (size_t)max(S + W, (kTMax / 32) * m.d) * 8;
    return acc + (size_t)((m.G * m.d + 1) & ~1) * 4 + (size_t)m.G * m.d * 8;
}

size_t decode_workspace_bytes(const Dims& m, int R) {
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t U = m.units;
    return al(U * R * 4) * 2 + al(U * m.G * R * 4) + al(U * R * 4);
}

}  // namespace ems
