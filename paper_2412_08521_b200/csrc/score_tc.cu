// score_tc.cu -- the tcgen05/TMEM/TMA score pass for bf16, head_dim 128, L % 128 == 0.
//
// (P1) fwd_tc: causal FlashAttention forward, Q-stationary.  One CTA owns two
//      128-row query tiles ("slots") that share one KV head (two heads of a GQA
//      group, or two consecutive tiles when G == 1) and streams K/V tiles through
//      a 2-stage TMA ring, so every K/V tile read from L2 feeds two QK^T MMAs.
//      S_t = Q_t K^T (SS MMA, M=N=128, K=128) lands in TMEM; the softmax of each
//      slot is split over two warpgroups, one per 64-column half of every row
//      (thread = half a row), which halves the softmax latency that sits between
//      a slot's S MMA and its PV MMA.  The halves agree on the row max through a
//      shared-memory exchange + named barrier per tile; P = exp2(S*c - m_ref) uses a
//      lazily-updated reference max (O is rescaled only when the max grows by > 8
//      in log2 units), is written as packed bf16 over S, and the MMA warp
//      accumulates O_t += P_t V (TS MMA: A from TMEM, V MN-major from smem).  MMA
//      order S0 S1 | PV0 S0' | PV1 S1' | ... keeps the tensor core on one slot
//      while the other slot's softmax runs.  Outputs: O (bf16), the negated row LSE
//      in log2 units (workspace, feeds P2) and optionally the natural-log LSE.
//
// (P2) colsum_tc.cu: KV-stationary column sums (glo, loc) normalised with P1's LSE.
//
// Reference semantics: streaming_pass, proj/src/scoring.cpp:20-64.
#include <cuda.h>
#include <stdlib.h>

#include "score_tc.cuh"
#include "tmap.h"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr float kRescaleThresh = 8.0f;  // log2 units

struct FwdArgs {
    int L, Hq, Hkv, G, nT;         // nT = L / 128
    int units;
    float c;                       // log2(e) / sqrt(d)
    __nv_bfloat16* out;            // [B*Hq][L][128] (may be null)
    float* nlse2;                  // [B*Hq][L] negated log2-domain LSE (always)
    float* lse_nat;                // [B*Hq][L] natural LSE (may be null)
    int unit_major;                // CTA order: 1 = unit by unit (L2 reuse of K/V), 0 = tile-major
};

constexpr int kFwdStages = 2;
// w0 TMA, w1 MMA; softmax warps 2..17: slot t = (w-2)/8, column half
// h = ((w-2)/4) % 2, TMEM sub-partition w % 4.
constexpr int kFwdThreads = 576;
constexpr size_t kFwdSmem = 1024 + (2 + 2 * kFwdStages) * kTileBytes + 2 * 2 * 2 * 128 * 4;

struct FwdBars {
    uint64_t q_full;
    uint64_t k_full[kFwdStages], v_full[kFwdStages], kv_empty[kFwdStages];
    uint64_t s_full[2], p_full[2], o_full[2];
    uint32_t tmem_base;
};

// Work item -> (plane of slot 0, plane of slot 1, tile of slot 0, tile of slot 1, unit)
__device__ __forceinline__ void fwd_item(const FwdArgs& a, int bid, int& plane0, int& plane1,
                                         int& tile0, int& tile1, int& unit) {
    if (a.G >= 2) {
        const int pairs = a.G / 2;
        int I, hp;
        if (a.unit_major) {  // units in order, heaviest tiles first within a unit (K/V stay in L2)
            const int per_unit = a.nT * pairs;
            unit = bid / per_unit;
            const int r = bid % per_unit;
            I = a.nT - 1 - r / pairs;
            hp = r % pairs;
        } else {
            const int per_tile = a.units * pairs;
            I = a.nT - 1 - bid / per_tile;  // heaviest tiles first
            const int rem = bid % per_tile;
            unit = rem / pairs;
            hp = rem % pairs;
        }
        const int b = unit / a.Hkv, hk = unit % a.Hkv;
        plane0 = b * a.Hq + hk * a.G + 2 * hp;
        plane1 = plane0 + 1;
        tile0 = tile1 = I;
    } else {
        const int npair = a.nT / 2;
        const int p = a.unit_major ? npair - 1 - bid % npair : npair - 1 - bid / a.units;
        unit = a.unit_major ? bid / npair : bid % a.units;
        const int b = unit / a.Hkv, hk = unit % a.Hkv;
        plane0 = plane1 = b * a.Hq + hk;  // G == 1: query head == kv head
        tile0 = 2 * p;
        tile1 = 2 * p + 1;
    }
}

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int kPoly>
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const __grid_constant__ CUtensorMap tv, const FwdArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sq = sm;                                  // 2 x 32 KB
    uint8_t* sk = sq + 2 * kTileBytes;                 // stages x 32 KB
    uint8_t* sv = sk + kFwdStages * kTileBytes;        // stages x 32 KB
    float* xch = reinterpret_cast<float*>(sv + kFwdStages * kTileBytes);  // [slot][buf][half][128]
    __shared__ FwdBars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    int plane[2], tile[2], unit;
    fwd_item(a, blockIdx.x, plane[0], plane[1], tile[0], tile[1], unit);
    const int jmax = max(tile[0], tile[1]);

    if (warp == 0) {
        tmem_alloc<512>(&bars.tmem_base);
    } else if (warp == 1 && elect_one()) {
        mbar_init(&bars.q_full, 1);
        for (int s = 0; s < kFwdStages; ++s) {
            mbar_init(&bars.k_full[s], 1);
            mbar_init(&bars.v_full[s], 1);
            mbar_init(&bars.kv_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bars.s_full[t], 1);
            mbar_init(&bars.p_full[t], 256);
            mbar_init(&bars.o_full[t], 1);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    // TMEM columns: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_t aliases S_t[0,64)
    const uint32_t tS[2] = {tmem, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 384};

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (elect_one()) {
            tma_prefetch(&tq);
            tma_prefetch(&tk);
            tma_prefetch(&tv);
            mbar_expect_tx(&bars.q_full, 2 * kTileBytes);
            for (int t = 0; t < 2; ++t) {
                uint8_t* dst = sq + t * kTileBytes;
                tma_load_3d(dst, &tq, &bars.q_full, 0, tile[t] * kTile, plane[t]);
                tma_load_3d(dst + 16384, &tq, &bars.q_full, 64, tile[t] * kTile, plane[t]);
            }
            for (int j = 0; j <= jmax; ++j) {
                const int s = j % kFwdStages;
                if (j >= kFwdStages) mbar_wait(&bars.kv_empty[s], ((j / kFwdStages) - 1) & 1);
                uint8_t* dk = sk + s * kTileBytes;
                uint8_t* dv = sv + s * kTileBytes;
                mbar_expect_tx(&bars.k_full[s], kTileBytes);
                tma_load_3d(dk, &tk, &bars.k_full[s], 0, j * kTile, unit);
                tma_load_3d(dk + 16384, &tk, &bars.k_full[s], 64, j * kTile, unit);
                mbar_expect_tx(&bars.v_full[s], kTileBytes);
                tma_load_3d(dv, &tv, &bars.v_full[s], 0, j * kTile, unit);
                tma_load_3d(dv + 16384, &tv, &bars.v_full[s], 64, j * kTile, unit);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t id_s = idesc_bf16(128, 128, 0, 0);   // Q (K-major) x K^T (K-major)
            const uint32_t id_o = idesc_bf16(128, 128, 0, 1);   // P (TMEM) x V (MN-major)
            auto issue_s = [&](int t, int j) {
                const int s = j % kFwdStages;
                const uint32_t qa = smem_u32(sq + t * kTileBytes);
                const uint32_t ka = smem_u32(sk + s * kTileBytes);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ss(tS[t], sdesc(kmajor_addr(qa, k), 16, 1024),
                           sdesc(kmajor_addr(ka, k), 16, 1024), id_s, k > 0);
                mma_commit(&bars.s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {
                const int s = j % kFwdStages;
                const uint32_t va = smem_u32(sv + s * kTileBytes);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ts(tO[t], tS[t] + k * 8, sdesc(va + k * 2048, 16384, 1024), id_o,
                           (j > 0 || k > 0) ? 1u : 0u);
                mma_commit(&bars.o_full[t]);
            };
            mbar_wait(&bars.q_full, 0);
            mbar_wait(&bars.k_full[0], 0);
            tc_fence_after();
            issue_s(0, 0);
            issue_s(1, 0);
            for (int j = 0; j <= jmax; ++j) {
                const int s = j % kFwdStages;
                const uint32_t sp = (j / kFwdStages) & 1;
                bool v_ready = false, k_next_ready = false;
                for (int t = 0; t < 2; ++t) {
                    if (j > tile[t]) continue;
                    mbar_wait(&bars.p_full[t], j & 1);
                    if (!v_ready) {
                        mbar_wait(&bars.v_full[s], sp);
                        v_ready = true;
                    }
                    tc_fence_after();
                    issue_pv(t, j);
                    if (j + 1 <= tile[t]) {
                        if (!k_next_ready) {
                            const int s1 = (j + 1) % kFwdStages;
                            mbar_wait(&bars.k_full[s1], ((j + 1) / kFwdStages) & 1);
                            k_next_ready = true;
                            tc_fence_after();
                        }
                        issue_s(t, j + 1);
                    }
                }
                mma_commit(&bars.kv_empty[s]);
            }
        }
    } else {
        // ---------------------------------------------------------------- softmax (half rows)
        const int t = (warp - 2) >> 3;          // slot
        const int h = ((warp - 2) >> 2) & 1;    // column half: keys [64h, 64h + 64)
        const int wi = warp & 3;                // TMEM sub-partition
        const int m = wi * 32 + (tid & 31);     // row within the tile
        const int I = tile[t];
        const uint32_t sS = tmem_lane_addr(tS[t], wi) + 64 * h;   // this thread's S half
        const uint32_t sP = tmem_lane_addr(tS[t], wi) + 32 * h;   // its packed-P half
        const uint32_t sO = tmem_lane_addr(tO[t], wi) + 64 * h;   // its O half
        float* xt = xch + t * 2 * 2 * 128;      // [buf][half][128]
        const int bar_id = 1 + t;
        float m_ref = -INFINITY, l = 0.f;
        for (int j = 0; j <= I; ++j) {
            mbar_wait(&bars.s_full[t], j & 1);
            tc_fence_after();
            uint32_t r[2][32];
            tmem_ld32(sS, r[0]);
            tmem_ld32(sS + 32, r[1]);
            tmem_ld_wait();
            if (j == I) {  // diagonal tile: key 64h + n > query m is masked
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int x = 0; x < 32; ++x)
                        if (64 * h + c * 32 + x > m) r[c][x] = __float_as_uint(-INFINITY);
            }
            // half-row max: 3-input FMNMX3, four independent chains
            float hmv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int x = 0; x < 32; x += 8)
#pragma unroll
                    for (int g = 0; g < 4; g += 2) {
                        hmv[g] = fmax3(hmv[g], __uint_as_float(r[c][x + 2 * g]), __uint_as_float(r[c][x + 2 * g + 1]));
                        hmv[g + 1] = fmax3(hmv[g + 1], __uint_as_float(r[c][x + 2 * g + 2]),
                                           __uint_as_float(r[c][x + 2 * g + 3]));
                    }
            const float hm = fmax3(hmv[0], hmv[1], fmaxf(hmv[2], hmv[3]));
            // exchange half-row maxima (also orders both halves' S loads before any P store,
            // since P of half 1 overwrites S columns 32..63 of half 0)
            float* xb = xt + (j & 1) * 256;
            const uint32_t xs = smem_u32(xb);  // explicit shared ops (generic LD/ST stall here)
            sts32(xs + 4 * (h * 128 + m), hm);
            named_sync(bar_id, 256);
            const float mx = fmaxf(hm, lds32(xs + 4 * ((h ^ 1) * 128 + m)));
            const float mx2 = mx * a.c;
            const bool need = mx2 > m_ref + kRescaleThresh;
            const bool warp_need = __any_sync(0xffffffffu, need);
            const float new_m = need ? mx2 : m_ref;
            const float corr = need ? ex2(m_ref - new_m) : 1.f;
            m_ref = new_m;
            l *= corr;
            const float2 c2 = make_float2(a.c, a.c), nm2 = make_float2(-m_ref, -m_ref);
            float2 rs2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    const float2 arg = __ffma2_rn(
                        make_float2(__uint_as_float(r[c][2 * x]), __uint_as_float(r[c][2 * x + 1])), c2, nm2);
                    float2 p;
                    if ((x & 7) < kPoly) p = ex2_poly2(arg);
                    else p = make_float2(ex2(arg.x), ex2(arg.y));
                    rs2 = __fadd2_rn(rs2, p);
                    pk[x] = pack_bf16(p.x, p.y);
                }
                tmem_st16(sP + c * 16, pk);
            }
            l += rs2.x + rs2.y;
            if (warp_need && j > 0) {  // rescale this half of O_t once PV(j-1) has landed (rare)
                mbar_wait(&bars.o_full[t], (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t o[32];
                    tmem_ld32(sO + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int x = 0; x < 32; ++x) o[x] = __float_as_uint(__uint_as_float(o[x]) * corr);
                    tmem_st32(sO + c * 32, o);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&bars.p_full[t]);
        }
        // epilogue: l = l_half0 + l_half1 (fixed order), O / l -> bf16, LSE
        float* xb = xt + ((I + 1) & 1) * 256;
        const uint32_t xs = smem_u32(xb);
        sts32(xs + 4 * (h * 128 + m), l);
        named_sync(bar_id, 256);
        const float lt = h == 0 ? l + lds32(xs + 4 * (128 + m)) : lds32(xs + 4 * m) + l;
        mbar_wait(&bars.o_full[t], I & 1);
        tc_fence_after();
        const size_t row = (size_t)plane[t] * a.L + (size_t)I * kTile + m;
        const float inv = 1.f / lt;
        if (a.out) {
            uint4* dst = reinterpret_cast<uint4*>(a.out + row * kD + 64 * h);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                uint32_t o[32];
                tmem_ld32(sO + c * 32, o);
                tmem_ld_wait();
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    uint4 v;
                    v.x = pack_bf16(__uint_as_float(o[8 * x + 0]) * inv, __uint_as_float(o[8 * x + 1]) * inv);
                    v.y = pack_bf16(__uint_as_float(o[8 * x + 2]) * inv, __uint_as_float(o[8 * x + 3]) * inv);
                    v.z = pack_bf16(__uint_as_float(o[8 * x + 4]) * inv, __uint_as_float(o[8 * x + 5]) * inv);
                    v.w = pack_bf16(__uint_as_float(o[8 * x + 6]) * inv, __uint_as_float(o[8 * x + 7]) * inv);
                    dst[c * 4 + x] = v;
                }
            }
        }
        if (h == 0) {
            const float lse2 = m_ref + __log2f(lt);
            a.nlse2[row] = -lse2;  // negated: P2 computes s*c + nlse2 with one FFMA
            if (a.lse_nat) a.lse_nat[row] = lse2 * kLn2;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int kPoly>
void fwd_launch(int grid, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                const FwdArgs& fa, cudaStream_t s) {
    static const bool attr = [] {  // once per process, thread-safe (magic static)
        cudaFuncSetAttribute(fwd_tc_kernel<kPoly>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kFwdSmem);
        return true;
    }();
    (void)attr;
    fwd_tc_kernel<kPoly><<<grid, kFwdThreads, kFwdSmem, s>>>(tq, tk, tv, fa);
}

}  // namespace

bool score_tc_supported(const Dims& dm, int dtype) {
    if (dtype != EMS_BF16 || dm.d != kD || dm.L % kTile != 0) return false;
    if (dm.G == 1 && (dm.L / kTile) % 2 != 0) return false;
    if (dm.G > 1 && dm.G % 2 != 0) return false;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0 && encode_fn() != nullptr;
}

// workspace: nlse2 [B*Hq][L] fp32, then (head split only) fp64 partials [2][units][hsplit][L]
static size_t nlse2_bytes(const Dims& dm) {
    return (sizeof(float) * (size_t)dm.B * dm.Hq * dm.L + 255) / 256 * 256;
}
static size_t part_bytes(const Dims& dm) {
    const int hs = colsum_hsplit(dm.G, dm.L / kTile, dm.units);
    return hs > 1 ? 2 * sizeof(double) * (size_t)dm.units * hs * dm.L : 0;
}
size_t score_tc_workspace(const Dims& dm) {
    return nlse2_bytes(dm) + part_bytes(dm) + (fwd2_workspace(dm.units, dm.L) + 255) / 256 * 256;
}

cudaError_t score_tc(const Dims& dm, const void* q, const void* k, const void* v, void* o,
                     float* lse, float* glo, float* loc, void* ws, cudaStream_t s) {
    const int planes_q = dm.B * dm.Hq, planes_kv = dm.B * dm.Hkv;
    CUtensorMap tq, tk, tv;
    if (!make_tmap_bf16_3d(&tq, q, kD, dm.L, planes_q, kTile) ||
        !make_tmap_bf16_3d(&tk, k, kD, dm.L, planes_kv, kTile) ||
        !make_tmap_bf16_3d(&tv, v ? v : k, kD, dm.L, planes_kv, kTile))
        return cudaErrorInvalidValue;
    float* nlse2 = static_cast<float*>(ws);
    FwdArgs fa;
    fa.L = dm.L;
    fa.Hq = dm.Hq;
    fa.Hkv = dm.Hkv;
    fa.G = dm.G;
    fa.nT = dm.L / kTile;
    fa.units = dm.units;
    fa.c = kLog2e / sqrtf((float)kD);
    fa.out = static_cast<__nv_bfloat16*>(o);
    fa.nlse2 = nlse2;
    fa.lse_nat = lse;
    static const int unit_major = [] {
        const char* e = getenv("EMS_UNIT_MAJOR");  // tuning override
        return e ? atoi(e) : 1;
    }();
    fa.unit_major = unit_major;
    const int n_fwd = dm.G >= 2 ? fa.nT * dm.units * (dm.G / 2) : (fa.nT / 2) * dm.units;
    // pairs (of every 8) whose exp2 runs on the FMA pipe; EMS_P1_POLY overrides (tuning)
    static const int poly = [] {
        const char* e = getenv("EMS_P1_POLY");
        return e ? atoi(e) : 0;
    }();
    // P1 variant: 2 = CTA-pair kernel with 256-key tiles (fwd2_tc.cu, default: 4% faster and
    // 3% less energy per step on config 3), 1 = the single-CTA two-slot kernel above
    static const int p1 = [] {
        const char* e = getenv("EMS_P1_IMPL");
        return e ? atoi(e) : 2;
    }();
    if (p1 == 2 && fwd2_tc_supported(dm.G, fa.nT)) {
        float* kmax = reinterpret_cast<float*>(static_cast<char*>(ws) + nlse2_bytes(dm) + part_bytes(dm));
        cudaError_t e = launch_fwd2_tc(dm.L, dm.Hq, dm.Hkv, dm.G, dm.units, fa.c, o, nlse2, lse, tq, tk, tv, k,
                                       kmax, s, q);
        if (e != cudaSuccess) return e;
    } else
    switch (poly) {
        case 1: fwd_launch<1>(n_fwd, tq, tk, tv, fa, s); break;
        case 2: fwd_launch<2>(n_fwd, tq, tk, tv, fa, s); break;
        case 3: fwd_launch<3>(n_fwd, tq, tk, tv, fa, s); break;
        default: fwd_launch<0>(n_fwd, tq, tk, tv, fa, s); break;
    }
    ColArgs ca;
    ca.L = dm.L;
    ca.Hq = dm.Hq;
    ca.Hkv = dm.Hkv;
    ca.G = dm.G;
    ca.nT = fa.nT;
    ca.units = dm.units;
    ca.lwin = dm.lwin_scores;
    ca.c = fa.c;
    ca.nlse2 = nlse2;
    ca.glo = glo;
    ca.loc = loc;
    static const int p2_debug = [] {
        const char* e = getenv("EMS_P2_DEBUG");  // profiling experiments only
        return e ? atoi(e) : 0;
    }();
    ca.debug = p2_debug;
    ca.hsplit = colsum_hsplit(dm.G, fa.nT, dm.units);
    // P2 keeps the global heaviest-first order: unit by unit leaves the last unit's heaviest
    // key-tile pairs (the longest CTAs) to the end of the grid (measured +5% P2 time)
    static const int p2_unit_major = [] {
        const char* e = getenv("EMS_P2_UNIT_MAJOR");  // tuning override
        return e ? atoi(e) : 0;
    }();
    ca.unit_major = p2_unit_major;
    // P2 variant: 2 = CTA-pair (cta_group::2, M = N = 256) kernel, 1 = single-CTA kernel
    static const int p2 = [] {
        const char* e = getenv("EMS_P2_IMPL");
        return e ? atoi(e) : 1;
    }();
    if (ca.hsplit > 1) {
        ca.part_g = reinterpret_cast<double*>(static_cast<char*>(ws) + nlse2_bytes(dm));
        ca.part_l = ca.part_g + (size_t)dm.units * ca.hsplit * dm.L;
    }
    if (p2 == 2 && ca.hsplit == 1) return launch_colsum2_tc(ca, tk, tq, s);
    return launch_colsum_tc(ca, tk, tq, s);
}

}  // namespace ems
