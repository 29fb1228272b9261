// colsum_tc.cu -- (P2) KV-stationary column sums of the causal softmax, the
// Global-Local score of EMS ("modifying the loop order").
//
//   glo_j = (1/G) sum_h sum_{i >= j} P^h_ij ,  loc_j = (1/G) sum_h sum_{i >= L-w} P^h_ij
//   P^h_ij = exp2(q_i.k_j * c - lse2^h_i)   (exactly normalised with P1's row LSE)
// Reference semantics: streaming_pass column scatter, proj/src/scoring.cpp:52-62;
// GQA mean per contract D2.
//
// One CTA owns TWO 128-key tiles (J0 = 2*jp, J1 = J0 + 1) of one unit, both resident
// in smem, and streams every (query head h, query tile I >= J0) through a 4-stage
// TMA ring.  Each streamed Q tile feeds two SS MMAs  S^T_w = K_Jw Q_I^T  (keys on
// TMEM lanes), which halves the L2 traffic per MMA compared with one key tile per
// CTA (v1 was L2-bandwidth bound).  Warpgroup w owns key tile Jw: thread m owns key
// Jw*128 + m and the column sum over the 128 queries is an in-thread row sum.
// Interior tiles take a mask-free path where kPoly of every 8 exp2 pairs run as a
// degree-5 polynomial on the FMA pipe (ex2_poly2) and the rest on MUFU.  Per-item
// fp32 sums are accumulated in fp64 in item order -> deterministic.
#include <stdlib.h>

#include "score_tc.cuh"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr int kQStages = 4;
constexpr int kBufs = 2;                 // TMEM: 2 x (2 key tiles x 128 cols) = 512 cols
constexpr int kThreads = 384;            // w0 TMA, w1 MMA, w4-7 key tile J0, w8-11 key tile J1
constexpr size_t kSmem = 1024 + (2 + kQStages) * kTileBytes + kBufs * 512;

struct Bars {
    uint64_t k_full;
    uint64_t q_full[kQStages], q_empty[kQStages];
    uint64_t s_full[kBufs], s_empty[kBufs], l_full[kBufs];
    uint32_t tmem_base;
};

// Process one 128-query row of S^T for the thread's key (general path: masks).
__device__ __forceinline__ void row_masked(uint32_t sa, uint32_t lb, float c, int I, int Jw,
                                           int mrow, int loc_start, float& sg, float& sl) {
    const bool diag = (I == Jw);
    sg = 0.f;
    sl = 0.f;
#pragma unroll 1
    for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t r[2][32];
        tmem_ld32(sa + h2 * 64, r[0]);
        tmem_ld32(sa + h2 * 64 + 32, r[1]);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int c0 = (2 * h2 + cc) * 32;
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                const int n = c0 + x;
                float p = ex2(fmaf(__uint_as_float(r[cc][x]), c, lds32(lb + 4 * n)));
                if (diag && n < mrow) p = 0.f;  // query < key: masked
                sg += p;
                if (I * kTile + n >= loc_start) sl += p;
            }
        }
    }
}

template <int kPoly>
__device__ __forceinline__ float row_fast(uint32_t sa, uint32_t lb, float c) {
    const float2 c2 = make_float2(c, c);
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t r[2][32];
        tmem_ld32(sa + h2 * 64, r[0]);
        tmem_ld32(sa + h2 * 64 + 32, r[1]);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const uint32_t lc = lb + (2 * h2 + cc) * 128;
            float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
            for (int x = 0; x < 32; x += 4) {
                const float4 lv = lds128(lc + 4 * x);
                const float2 a0 = __ffma2_rn(
                    make_float2(__uint_as_float(r[cc][x]), __uint_as_float(r[cc][x + 1])), c2,
                    make_float2(lv.x, lv.y));
                const float2 a1 = __ffma2_rn(
                    make_float2(__uint_as_float(r[cc][x + 2]), __uint_as_float(r[cc][x + 3])), c2,
                    make_float2(lv.z, lv.w));
                const int e0 = x / 2, e1 = x / 2 + 1;
                float2 p0, p1;
                if ((e0 & 7) < kPoly) p0 = ex2_poly2(a0);
                else p0 = make_float2(ex2(a0.x), ex2(a0.y));
                if ((e1 & 7) < kPoly) p1 = ex2_poly2(a1);
                else p1 = make_float2(ex2(a1.x), ex2(a1.y));
                s0 = __fadd2_rn(s0, p0);
                s1 = __fadd2_rn(s1, p1);
            }
            acc = __fadd2_rn(acc, __fadd2_rn(s0, s1));
        }
    }
    return acc.x + acc.y;
}

template <int kPoly>
__global__ void __launch_bounds__(kThreads, 1)
    colsum_tc_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tq,
                     const ColArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sk = sm;                                  // K_J0 | K_J1 (2 x 32 KB)
    uint8_t* sq = sk + 2 * kTileBytes;                 // Q ring
    float* slse = reinterpret_cast<float*>(sq + kQStages * kTileBytes);  // [kBufs][128]
    __shared__ Bars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int jp = blockIdx.x / a.units;               // key-tile pair, heaviest first
    const int unit = blockIdx.x % a.units;
    const int b = unit / a.Hkv, hk = unit % a.Hkv;
    const int J0 = 2 * jp;
    const bool has1 = J0 + 1 < a.nT;
    const int span = a.nT - J0;
    const int n_items = a.G * span;                    // item i -> head i / span, tile J0 + i % span

    if (warp == 0) {
        tmem_alloc<512>(&bars.tmem_base);
    } else if (warp == 1 && elect_one()) {
        mbar_init(&bars.k_full, 1);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&bars.q_full[s], 1);
            mbar_init(&bars.q_empty[s], 1);
        }
        for (int s = 0; s < kBufs; ++s) {
            mbar_init(&bars.s_full[s], 1);
            mbar_init(&bars.s_empty[s], 256);
            mbar_init(&bars.l_full[s], 1);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------- TMA producer
        if (elect_one()) {
            tma_prefetch(&tk);
            tma_prefetch(&tq);
            mbar_expect_tx(&bars.k_full, (has1 ? 2 : 1) * kTileBytes);
            tma_load_3d(sk, &tk, &bars.k_full, 0, J0 * kTile, unit);
            tma_load_3d(sk + 16384, &tk, &bars.k_full, 64, J0 * kTile, unit);
            if (has1) {
                tma_load_3d(sk + kTileBytes, &tk, &bars.k_full, 0, (J0 + 1) * kTile, unit);
                tma_load_3d(sk + kTileBytes + 16384, &tk, &bars.k_full, 64, (J0 + 1) * kTile, unit);
            }
            for (int i = 0; i < n_items; ++i) {
                const int h = i / span, I = J0 + i % span;
                const int plane = b * a.Hq + hk * a.G + h;
                const int s = i % kQStages, bb = i % kBufs;
                if (i >= kQStages) mbar_wait(&bars.q_empty[s], ((i / kQStages) - 1) & 1);
                uint8_t* dq = sq + s * kTileBytes;
                mbar_expect_tx(&bars.q_full[s], kTileBytes);
                tma_load_3d(dq, &tq, &bars.q_full[s], 0, I * kTile, plane);
                tma_load_3d(dq + 16384, &tq, &bars.q_full[s], 64, I * kTile, plane);
                if (i >= kBufs) mbar_wait(&bars.s_empty[bb], ((i / kBufs) - 1) & 1);
                mbar_expect_tx(&bars.l_full[bb], 512);
                bulk_load(slse + bb * 128, a.nlse2 + (size_t)plane * a.L + (size_t)I * kTile, 512,
                          &bars.l_full[bb]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t id_s = idesc_bf16(128, 128, 0, 0);  // K (K-major) x Q^T (K-major)
            const uint32_t ka0 = smem_u32(sk), ka1 = smem_u32(sk + kTileBytes);
            mbar_wait(&bars.k_full, 0);
            for (int i = 0; i < n_items; ++i) {
                const int I = J0 + i % span;
                const int s = i % kQStages, bb = i % kBufs;
                mbar_wait(&bars.q_full[s], (i / kQStages) & 1);
                if (i >= kBufs) mbar_wait(&bars.s_empty[bb], ((i / kBufs) - 1) & 1);
                tc_fence_after();
                const uint32_t qa = smem_u32(sq + s * kTileBytes);
                const uint32_t d0 = tmem + bb * 256;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ss(d0, sdesc(kmajor_addr(ka0, k), 16, 1024), sdesc(kmajor_addr(qa, k), 16, 1024),
                           id_s, k > 0);
                if (has1 && I >= J0 + 1) {  // key tile J1 is fully masked against query tile J0
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_ss(d0 + 128, sdesc(kmajor_addr(ka1, k), 16, 1024),
                               sdesc(kmajor_addr(qa, k), 16, 1024), id_s, k > 0);
                }
                mma_commit(&bars.s_full[bb]);
                mma_commit(&bars.q_empty[s]);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------- column sums
        const int w = (warp - 4) >> 2;          // key tile J0 + w
        const int wi = warp & 3;
        const int mrow = wi * 32 + (tid & 31);  // key within the tile
        const int Jw = J0 + w;
        const bool active = (w == 0) || has1;
        const int loc_start = a.L - a.lwin;
        const int last_interior = (loc_start / kTile) - 1;  // tiles <= this hold no window query
        double acc_g = 0.0, acc_l = 0.0;
        for (int i = 0; i < n_items; ++i) {
            const int I = J0 + i % span;
            const int bb = i % kBufs;
            const uint32_t ph = (i / kBufs) & 1;
            mbar_wait(&bars.l_full[bb], ph);
            mbar_wait(&bars.s_full[bb], ph);
            tc_fence_after();
            if (active && I >= Jw) {
                const uint32_t sa = tmem_lane_addr(tmem + bb * 256 + w * 128, wi);
                const uint32_t lb = smem_u32(slse + bb * 128);
                if (I > Jw && I <= last_interior) {
                    acc_g += (double)row_fast<kPoly>(sa, lb, a.c);
                } else {
                    float sg, sl;
                    row_masked(sa, lb, a.c, I, Jw, mrow, loc_start, sg, sl);
                    acc_g += (double)sg;
                    acc_l += (double)sl;
                }
            }
            tc_fence_before();
            mbar_arrive(&bars.s_empty[bb]);
        }
        if (active) {
            const size_t o = (size_t)unit * a.L + (size_t)Jw * kTile + mrow;
            a.glo[o] = (float)(acc_g / a.G);
            a.loc[o] = (float)(acc_l / a.G);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int kPoly>
cudaError_t launch_t(const ColArgs& a, const CUtensorMap& tk, const CUtensorMap& tq, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(colsum_tc_kernel<kPoly>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kSmem);
        attr = true;
    }
    const dim3 grid(((a.nT + 1) / 2) * a.units);
    colsum_tc_kernel<kPoly><<<grid, kThreads, kSmem, s>>>(tk, tq, a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_colsum_tc(const ColArgs& a, const CUtensorMap& tk, const CUtensorMap& tq,
                             cudaStream_t s) {
    // pairs (of every 8) whose exp2 runs on the FMA pipe; EMS_P2_POLY overrides (tuning)
    static const int poly = [] {
        const char* e = getenv("EMS_P2_POLY");
        return e ? atoi(e) : 3;
    }();
    switch (poly) {
        case 0: return launch_t<0>(a, tk, tq, s);
        case 2: return launch_t<2>(a, tk, tq, s);
        case 4: return launch_t<4>(a, tk, tq, s);
        default: return launch_t<3>(a, tk, tq, s);
    }
}

}  // namespace ems
